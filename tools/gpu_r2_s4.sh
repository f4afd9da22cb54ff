mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_gmres_c4.csv python tools/gmres_big.py c4 50 1e-4 40 > gpurun_out/ncu_gm.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_gmres_c4.csv
