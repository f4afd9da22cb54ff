mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_reduced.py tests/test_gpu_precond.py -q -m gpu -x > gpurun_out/pytest_s6.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_s6.log
timeout 300 python tools/gmres_big.py c4 50 1e-4 200
timeout 600 python tools/reduced_big.py c4 4
timeout 600 python tools/reduced_big.py c3 4
