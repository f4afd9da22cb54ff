# Fused all-to-all pack/unpack in the slab y passes; full-size matvec parity from the oracle-written goldens.
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests/test_slab.py -m gpu -x -q --durations=8 ) > gpurun_out/pytest_slab_d3.log 2>&1; echo "slab rc=$?"; tail -14 gpurun_out/pytest_slab_d3.log
( time timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_size" --durations=8 ) > gpurun_out/pytest_full_d3.log 2>&1; echo "full rc=$?"; tail -14 gpurun_out/pytest_full_d3.log
for f in 1 0; do
AIM_SLAB_FUSE_PACK=$f timeout 600 python bench.py --slab --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-extra > gpurun_out/bench_slab_c4_fuse$f.json 2> gpurun_out/bench_slab_c4_fuse$f.err; echo "slab bench fuse=$f rc=$?"; cut -c1-400 gpurun_out/bench_slab_c4_fuse$f.json
done
