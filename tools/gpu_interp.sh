mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "interp_mma or nrhs or small" 2>&1 | tail -3
for rb in 8 16; do AIM_INTERP_RB=$rb timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ib$rb.json 2> gpurun_out/bench.err; echo "bench rc=$? rb=$rb"; tail -2 gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench_ib$rb.json')); print(d['value'], {k: round(v*1e3) for k,v in d['stage_ms'].items()})"; done
