# ncu --set full of the C4 product's kernels at the final HEAD (general path), incl. the fused mode-2 and x passes.
mkdir -p gpurun_out
timeout 300 python tools/prof_matvec.py c4 2 > gpurun_out/plain_d8.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'near1|project1|interp1i|phi_interleave|ymode2|fft_ct' -s 7 -c 7 \
  -o gpurun_out/prof_c4_d8 python tools/prof_matvec.py c4 2 > gpurun_out/ncu_full_c4_d8.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out/prof_c4_d8.ncu-rep
