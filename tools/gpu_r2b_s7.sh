# default bench line + launch list of the bench command + ncu --set full of the new kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_s17.json 2> gpurun_out/bench_s17.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_s17.err; cut -c1-600 gpurun_out/bench_s17.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_bench_s17.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_bench.log 2>&1; echo "ncu launch rc=$?"
python tools/launches.py gpurun_out/launches_bench_s17.csv > gpurun_out/launches_bench_s17.txt; tail -12 gpurun_out/launches_bench_s17.txt
timeout 300 python tools/prof_matvec.py c4 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'interp1i|phi_interleave|near1|project1' -s 4 -c 4 \
  -o gpurun_out/prof_c4_s17 python tools/prof_matvec.py c4 2 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu full rc=$?"
timeout 300 python tools/prof_matvec.py c4 2 cmp > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'cp_spmm|near_spmm|cp_gather_sum|interp1i' -s 6 -c 4 \
  -o gpurun_out/prof_c4cmp_s17 python tools/prof_matvec.py c4 2 cmp > gpurun_out/ncu_full_c4cmp.log 2>&1; echo "ncu full cmp rc=$?"
ls -la gpurun_out/*.ncu-rep
