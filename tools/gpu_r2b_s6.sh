# one coefficient fetch per GMRES iteration; compressed near SpMM retiled; interleaved-potential interpolation
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_parity.py -q -x -k "gmres or compressed or stages or matvec_small or full_size_sampled_rows" > gpurun_out/pytest_b6.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_b6.log
timeout 600 python tools/cmp_quick.py c4 50 > gpurun_out/cmp_c4f.json 2> gpurun_out/cmp_c4f.err; echo "cmp rc=$?"; tail -3 gpurun_out/cmp_c4f.err; cat gpurun_out/cmp_c4f.json
AIM_INTERP_IL=0 timeout 600 python tools/cmp_quick.py c4 > gpurun_out/cmp_c4f_noil.json 2>&1; echo "cmp noil"; cut -c1-300 gpurun_out/cmp_c4f_noil.json
timeout 600 python tools/cmp_quick.py c5 > gpurun_out/cmp_c5f.json 2> gpurun_out/cmp_c5f.err; echo "cmp rc=$?"; cat gpurun_out/cmp_c5f.json
timeout 600 python tools/cmp_quick.py c3 > gpurun_out/cmp_c3f.json 2> gpurun_out/cmp_c3f.err; echo "cmp rc=$?"; cut -c1-400 gpurun_out/cmp_c3f.json
timeout 300 python tools/prof_matvec.py c4 3 cmp > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4_cmp.csv python tools/prof_matvec.py c4 3 cmp > gpurun_out/ncu_cmp.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_c4_cmp.csv | grep -v "weights\|proj_\|kernel_sample\|spectrum\|near_scan\|near_sort\|htab\|near_values" | tee gpurun_out/launches_c4_cmp.txt
