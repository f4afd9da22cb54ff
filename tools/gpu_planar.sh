mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_slab.py -m gpu -x -q -k "stages or small or nrhs or c2_full or spectrum or slab_matvec_vs" 2>&1 | tail -3
for k in default stockham; do AIM_PLANAR_KERNEL=$k timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pl_$k.json 2> gpurun_out/bench.err; echo "bench rc=$? $k"; tail -2 gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench_pl_$k.json')); print(d['value'], {k: round(v*1e3) for k,v in d['stage_ms'].items()})"; done
