mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "host_steps or host_pipeline or matvec_small or gmres_c1" > gpurun_out/pytest_s1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_s1.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_s1.json 2> gpurun_out/bench_s1.err; echo "bench rc=$?"; tail -5 gpurun_out/bench_s1.err; cat gpurun_out/bench_s1.json
