# Why does the lean 16-byte kernel win in bench.py (eager launches, 2^28) and lose slightly
# in gpubench (graph replays of one kernel, 2^27)?  Same A/B across size, graph timing and PDL.
mkdir -p gpurun_out
o=gpurun_out/v16_ab2.txt; : > $o
fmt='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print("value %.2f G  " % (d["value"]/1e9) + "  ".join("%s %.0f" % (k, v["gbs"]) for k, v in d["per_op"].items()) + "  sm_mhz %s" % d["clocks"]["sm_mhz"])'
B="python bench.py --no-sub-workloads --no-e2e --no-cpu-baseline --no-check --no-device-batch --steps 20 --warmup 5"
for r in 1 2; do
  for v in 0 all; do
    export TF_EW_V16=$v
    echo -n "v16=$v eager 2^27  " >> $o; timeout 600 $B --elems 134217728 2>/dev/null | python -c "$fmt" >> $o
    echo -n "v16=$v graph 2^28  " >> $o; timeout 600 $B --graph on 2>/dev/null | python -c "$fmt" >> $o
    echo -n "v16=$v graph 2^27  " >> $o; timeout 600 $B --graph on --elems 134217728 2>/dev/null | python -c "$fmt" >> $o
    echo -n "v16=$v nopdl 2^28  " >> $o; TF_PDL=0 timeout 600 $B 2>/dev/null | python -c "$fmt" >> $o
  done
done
unset TF_EW_V16
echo done >> $o
