mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stages or small or nrhs or c64" 2>&1 | tail -3
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], {k: round(v*1e3) for k,v in d['stage_ms'].items()})"
timeout 900 python tools/try_big.py c3 c4 c5 2>&1 | cut -c1-600
