# Round-2 closing check at HEAD: smoke, the whole gpu suite, the default bench line (own arm and reference arm).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_d1.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_d1.log
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/pytest_gpu_d1.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_gpu_d1.log
( time timeout 900 python bench.py ) > gpurun_out/bench_d1.json 2> gpurun_out/bench_d1.err; echo "bench rc=$?"; tail -4 gpurun_out/bench_d1.err; cut -c1-1500 gpurun_out/bench_d1.json
( time timeout 600 python bench.py --impl reference --steps 2 --warmup 1 ) > gpurun_out/bench_ref_d1.json 2> gpurun_out/bench_ref_d1.err; echo "ref rc=$?"; tail -4 gpurun_out/bench_ref_d1.err; cut -c1-800 gpurun_out/bench_ref_d1.json
