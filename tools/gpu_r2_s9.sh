mkdir -p gpurun_out
timeout 300 python tools/prof_matvec.py c4 2 > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'ymode2|interp1|project1|near1' -s 4 -c 4 \
  -o gpurun_out/prof_c4_r2 python tools/prof_matvec.py c4 2 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full_c4.log
