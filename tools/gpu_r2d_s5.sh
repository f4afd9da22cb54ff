# Whole gpu suite at HEAD (full-size matvec parity from the oracle-written goldens, fused slab pack, C4 GMRES cycle), then bench.
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 ) > gpurun_out/pytest_gpu_d5.log 2>&1; echo "pytest rc=$?"; tail -24 gpurun_out/pytest_gpu_d5.log
( time timeout 900 python bench.py ) > gpurun_out/bench_d5.json 2> gpurun_out/bench_d5.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_d5.err; cut -c1-400 gpurun_out/bench_d5.json
