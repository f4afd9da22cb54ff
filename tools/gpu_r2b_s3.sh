# GMRES: fused last-block reductions, 3-stage axpy_dot pipeline, 2 elements per thread in axpy_norm
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_parity.py -q -x -k "gmres" > gpurun_out/pytest_b3.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_b3.log
timeout 600 python tools/cmp_quick.py c4 50 > gpurun_out/cmp_c4c.json 2> gpurun_out/cmp_c4c.err; echo "cmp rc=$?"; tail -3 gpurun_out/cmp_c4c.err; cat gpurun_out/cmp_c4c.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_gmres_c4c.csv python tools/gmres_big.py c4 50 1e-4 50 > gpurun_out/ncu_gm.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_gmres_c4c.csv | grep -E "mdot|axpy|scale|reduce|combine" | tee gpurun_out/launches_gmres_c4c.txt
