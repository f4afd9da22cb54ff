mkdir -p gpurun_out
timeout 300 python tools/gmres_big.py c4 50 1e-4 200 > gpurun_out/gmres_c4_200.log 2>&1; cat gpurun_out/gmres_c4_200.log
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_gmres.py tests/test_slab.py -q -m gpu -k "not c3 and not c4 and not c5" > gpurun_out/pytest_s3.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_s3.log
