mkdir -p gpurun_out
for c in c4 c5; do for v in off,prio256_nc prio256_fc prio128_fc off,prio128_nc; do
timeout 300 python tools/ovl_ab.py $c 50 $v > gpurun_out/prio_$c_$v.log 2>&1; echo "$c $v rc=$?"; tail -1 gpurun_out/prio_$c_$v.log | cut -c1-400; done; done
