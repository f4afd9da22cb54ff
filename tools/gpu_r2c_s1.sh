# near SpMV beside the FFT: parity tests, A/B on C4/C3/C5/C2, rank-local slab near rows
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "near_stream or rank_local" > gpurun_out/pytest_s1.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_s1.log
for c in c4 c3 c5; do timeout 600 python tools/ovl_ab.py $c 50 > gpurun_out/ovl_$c.log 2>&1; echo "ovl $c rc=$?"; tail -1 gpurun_out/ovl_$c.log; done
