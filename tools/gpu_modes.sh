mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_slab.py -m gpu -x -q -k "conv_modes or slab_matvec_vs or spectrum or stages" 2>&1 | tail -3
timeout 900 python tools/try_big.py c3 c4 c5 2>&1 | cut -c1-600
timeout 600 python tools/slab_try.py c4 4 2>&1 | tail -1
