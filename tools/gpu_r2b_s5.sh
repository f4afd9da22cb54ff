# GMRES: thread-per-element axpy_norm, axpy_dot at 3 CTAs/SM, next product enqueued before the host Givens;
# compressed products with the near field on the side stream
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_precond.py tests/test_gpu_parity.py -q -x -k "gmres or compressed or precond" > gpurun_out/pytest_b5.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_b5.log
timeout 600 python tools/cmp_quick.py c4 50 > gpurun_out/cmp_c4e.json 2> gpurun_out/cmp_c4e.err; echo "cmp rc=$?"; tail -3 gpurun_out/cmp_c4e.err; cat gpurun_out/cmp_c4e.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_gmres_c4e.csv python tools/gmres_big.py c4 50 1e-4 50 > gpurun_out/ncu_gm.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_gmres_c4e.csv | grep -E "mdot|axpy|scale|reduce|combine" | tee gpurun_out/launches_gmres_c4e.txt
