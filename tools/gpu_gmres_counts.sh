mkdir -p gpurun_out
for c in c2 c3 c5; do timeout 600 python tools/gmres_big.py $c 50 1e-4 20000; done > gpurun_out/gmres_counts.log 2>&1
cat gpurun_out/gmres_counts.log
