mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.txt 2>&1; cat gpurun_out/fp64_peak.txt
timeout 300 python tools/prof_matvec.py c2 3 > gpurun_out/plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'near_b4|planar_ct|fft_ct|project_kernel|interp_kernel' -s 11 -c 6 -o gpurun_out/prof_full python tools/prof_matvec.py c2 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
