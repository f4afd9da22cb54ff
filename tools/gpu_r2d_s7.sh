# Final check at HEAD: smoke, whole gpu suite, default bench.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_d7.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_d7.log
( time timeout 900 python bench.py ) > gpurun_out/bench_d7.json 2> gpurun_out/bench_d7.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_d7.err; cut -c1-300 gpurun_out/bench_d7.json
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/pytest_gpu_d7.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu_d7.log
