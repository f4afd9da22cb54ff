# Round-2 baseline on one B200: large-config timings + C4 launch list with DRAM bytes.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
timeout 600 python tools/try_big.py c4 c3 c5 > gpurun_out/big_r2base.log 2>&1; echo "try_big rc=$?"; cat gpurun_out/big_r2base.log
timeout 300 python tools/prof_matvec.py c4 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4.csv python tools/prof_matvec.py c4 2 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_c4.csv
