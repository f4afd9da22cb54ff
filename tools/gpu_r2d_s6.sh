# ymode2 with the zero-padding rows skipped in the first forward / last inverse stage: parity, then bench.
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mode2 or full_size or conv" --durations=5 ) > gpurun_out/pytest_ym2_d6.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_ym2_d6.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extra > gpurun_out/bench_d6.json 2> gpurun_out/bench_d6.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_d6.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["clocks"], json.dumps(d.get("stage_ms") or d.get("stages") or {k:v for k,v in d.items() if "stage" in k})[:600])
PY
