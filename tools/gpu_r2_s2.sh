mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_gmres.py tests/test_slab.py -x -q -m gpu -k "not c3 and not c4 and not c5" > gpurun_out/pytest_s2.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_s2.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gmres" >> gpurun_out/pytest_s2.log 2>&1; echo "pytest2 rc=$?"; tail -3 gpurun_out/pytest_s2.log
for c in c2 c3 c5 c4; do timeout 600 python tools/gmres_big.py $c 50 1e-4 20000 --precond; done > gpurun_out/gmres_pre.log 2>&1; cat gpurun_out/gmres_pre.log
timeout 300 python tools/gmres_big.py c4 50 1e-4 200 > gpurun_out/gmres_c4_200.log 2>&1; cat gpurun_out/gmres_c4_200.log
