# Bench several library builds (build/variants/lib_*.so) back to back.
mkdir -p gpurun_out
for v in "$@"; do
  AIM_LIB=$PWD/build/variants/lib_$v.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  echo "$v rc=$?"; tail -2 gpurun_out/bench_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$v.json'));print('$v', round(d['value']), {k: round(v*1e3) for k,v in d['stage_ms'].items()})"
done
