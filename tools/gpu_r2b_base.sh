# Re-entry check of HEAD on a B200: full gpu suite, smoke, default bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/pytest_gpu_b.log 2>&1; echo "pytest rc=$?"; tail -40 gpurun_out/pytest_gpu_b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench rc=$?"; tail -5 gpurun_out/bench_b.err; cut -c1-1500 gpurun_out/bench_b.json
