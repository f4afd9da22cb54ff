# Quick GPU check: selected gpu tests, then the bench (no cpu baseline) and a launch list.
# Usage (under gpurun): bash tools/gpu_quick2.sh "<pytest -k expr>"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
