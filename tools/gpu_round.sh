# One GPU round: gpu tests, bench, launch list (+dram), full ncu capture of the top kernels.
# Usage (under gpurun): bash tools/gpu_round.sh [config]
CFG=${1:-c2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python tools/prof_matvec.py $CFG 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/prof_matvec.py $CFG 3 > gpurun_out/ncu_launch.log 2>&1
python tools/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt; cat gpurun_out/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'near_mma|planar4|fft_ct|project_kernel|interp_kernel' \
  -s 8 -c 6 -o gpurun_out/prof_full python tools/prof_matvec.py $CFG 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
