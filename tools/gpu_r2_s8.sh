mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused_mode2 or conv_modes_forced" > gpurun_out/pytest_s8.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_s8.log
timeout 600 python tools/try_big.py c4 c3
AIM_YZ_FUSED=0 timeout 600 python tools/try_big.py c4 c3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "full_size_sampled" > gpurun_out/pytest_s8b.log 2>&1; echo "pytest full rc=$?"; tail -5 gpurun_out/pytest_s8b.log
