mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_slab.py -m gpu -x -q -k nccl 2>&1 | tail -2
timeout 600 python bench.py --slab --steps 20 --warmup 3 > gpurun_out/bench_slab_c4.json 2> gpurun_out/bench_slab.err; echo "slab bench rc=$?"; tail -3 gpurun_out/bench_slab.err; cat gpurun_out/bench_slab_c4.json | cut -c1-600
timeout 900 python tools/try_big.py c3 c4 c5 > gpurun_out/big.log 2>&1; cat gpurun_out/big.log | cut -c1-700
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline'])"
