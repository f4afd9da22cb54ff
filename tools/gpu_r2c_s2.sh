mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "near_stream or rank_local or slab or smoke or abi" > gpurun_out/pytest_s2.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_s2.log
timeout 600 python tools/ovl_ab.py c4 50 > gpurun_out/ovl_c4b.log 2>&1; echo "ovl rc=$?"; tail -1 gpurun_out/ovl_c4b.log
