# Time the near kernels of several library builds (build/variants/lib_*.so), plus an ncu capture of the first.
mkdir -p gpurun_out
for v in "$@"; do
  AIM_LIB=$PWD/build/variants/lib_$v.so timeout 300 python tools/near_bench.py c2 20 2>&1 | tee -a gpurun_out/near_variants.log
done
AIM_LIB=$PWD/build/variants/lib_$1.so AIM_NEAR_KERNEL=mma timeout 600 ncu --set full --clock-control none --import-source on -k regex:near_mma_kernel -s 2 -c 1 -o gpurun_out/prof_near python tools/near_bench.py c2 2 > gpurun_out/ncu_near.log 2>&1; echo "ncu rc=$?"
