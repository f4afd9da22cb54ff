# compressed projection/interpolation: parity + timing; GMRES with the fixed product input; ymode2 28x28 plan
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "compressed or fused_mode2" > gpurun_out/pytest_b1.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_b1.log
timeout 600 python tools/cmp_quick.py c4 50 > gpurun_out/cmp_c4.json 2> gpurun_out/cmp_c4.err; echo "cmp rc=$?"; tail -3 gpurun_out/cmp_c4.err; cat gpurun_out/cmp_c4.json
AIM_YM2_PLAN=3 timeout 600 python tools/cmp_quick.py c4 > gpurun_out/cmp_c4_p3.json 2> gpurun_out/cmp_c4_p3.err; echo "cmp p3 rc=$?"; cat gpurun_out/cmp_c4_p3.json
timeout 600 python tools/cmp_quick.py c5 > gpurun_out/cmp_c5.json 2> gpurun_out/cmp_c5.err; echo "cmp rc=$?"; cat gpurun_out/cmp_c5.json
timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_precond.py -q -x > gpurun_out/pytest_b1g.log 2>&1; echo "pytest gm rc=$?"; tail -5 gpurun_out/pytest_b1g.log
