# tiled TMA interpolation: parity + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "interp_tile or stages or matvec_small or compressed_projection" > gpurun_out/pytest_b4.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_b4.log
timeout 600 python tools/cmp_quick.py c4 > gpurun_out/cmp_c4d.json 2> gpurun_out/cmp_c4d.err; echo "cmp rc=$?"; tail -3 gpurun_out/cmp_c4d.err; cat gpurun_out/cmp_c4d.json
timeout 600 python tools/cmp_quick.py c5 > gpurun_out/cmp_c5d.json 2> gpurun_out/cmp_c5d.err; echo "cmp rc=$?"; tail -3 gpurun_out/cmp_c5d.err; cat gpurun_out/cmp_c5d.json
AIM_INTERP_TILE=0 timeout 600 python tools/cmp_quick.py c3 > gpurun_out/cmp_c3_notile.json 2>&1; cat gpurun_out/cmp_c3_notile.json | cut -c1-400
timeout 600 python tools/cmp_quick.py c3 > gpurun_out/cmp_c3d.json 2>&1; cat gpurun_out/cmp_c3d.json | cut -c1-400
