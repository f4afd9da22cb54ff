# element-batched compressed projection: parity + timing; GMRES pass breakdown (ncu launch list)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "compressed" > gpurun_out/pytest_b2.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_b2.log
timeout 600 python tools/cmp_quick.py c4 > gpurun_out/cmp_c4b.json 2> gpurun_out/cmp_c4b.err; echo "cmp rc=$?"; tail -3 gpurun_out/cmp_c4b.err; cat gpurun_out/cmp_c4b.json
timeout 600 python tools/cmp_quick.py c5 > gpurun_out/cmp_c5b.json 2> gpurun_out/cmp_c5b.err; echo "cmp rc=$?"; cat gpurun_out/cmp_c5b.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_gmres_c4b.csv python tools/gmres_big.py c4 50 1e-4 50 > gpurun_out/ncu_gm.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_gmres_c4b.csv | tee gpurun_out/launches_gmres_c4b.txt
