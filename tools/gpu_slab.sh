mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_slab.py -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --slab --steps 20 --warmup 3 > gpurun_out/bench_slab_c4.json 2> gpurun_out/bench_slab.err; echo "slab bench rc=$?"; tail -3 gpurun_out/bench_slab.err; cat gpurun_out/bench_slab_c4.json | cut -c1-900
timeout 600 python tools/slab_try.py c4 4 2>&1 | tail -1
