# ncu --set full of one kernel (regex $1) for each library variant ($2...)
mkdir -p gpurun_out
K=$1; shift
for v in "$@"; do
  AIM_LIB=$PWD/build/variants/lib_$v.so timeout 300 python tools/prof_matvec.py c2 2 > gpurun_out/plain_$v.log 2>&1 && \
  AIM_LIB=$PWD/build/variants/lib_$v.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
     -o gpurun_out/prof_$v python tools/prof_matvec.py c2 2 > gpurun_out/ncu_$v.log 2>&1
  echo "$v rc=$?"
done
