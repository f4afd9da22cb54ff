# Re-entry check at HEAD: gpu tests, smoke, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/pytest_gpu_c.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu_c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_c.log
timeout 900 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_c.err; cut -c1-800 gpurun_out/bench_c.json
