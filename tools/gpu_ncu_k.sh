# ncu --set full of one launch of kernels matching $1 in a c2 matvec run (skip $2 matching launches)
mkdir -p gpurun_out
timeout 300 python tools/prof_matvec.py c2 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-1} -c 1 -o gpurun_out/prof_$3 python tools/prof_matvec.py c2 3 > gpurun_out/ncu_k.log 2>&1
echo "ncu rc=$?"
