# ncu --set full of the first launch of kernels matching $1 in a c2 matvec run (library: default or $2)
mkdir -p gpurun_out
K=$1; OUT=${3:-prof_one}
[ -n "$2" ] && export AIM_LIB=$PWD/build/variants/lib_$2.so
timeout 300 python tools/prof_matvec.py c2 2 > gpurun_out/plain_one.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -c ${4:-1} -o gpurun_out/$OUT python tools/prof_matvec.py c2 2 > gpurun_out/ncu_one.log 2>&1
echo "ncu rc=$?"
