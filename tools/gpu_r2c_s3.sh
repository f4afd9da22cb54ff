mkdir -p gpurun_out
for c in c4 c3 c5; do timeout 600 python tools/ovl_ab.py $c 50 > gpurun_out/prio_$c.log 2>&1; echo "prio $c rc=$?"; tail -1 gpurun_out/prio_$c.log; done
