# The new C4 GMRES one-cycle test with its slow oracle leg, then the bench launch list at HEAD.
mkdir -p gpurun_out
( time AIM_TEST_SLOW=1 timeout 1500 python -m pytest tests/test_gpu_gmres.py -m gpu -x -q -k c4_one_cycle ) > gpurun_out/pytest_c4gm_d2.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_c4gm_d2.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_d2_plain.json 2> gpurun_out/bench_d2_plain.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_d2.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_d2.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_d2.csv > gpurun_out/launches_d2.txt; head -40 gpurun_out/launches_d2.txt
