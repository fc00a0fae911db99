# Lean 16-byte elementwise kernel (one 16-byte vector per plane per thread, <= 32
# registers, 8 CTAs/SM) vs the lean 32-byte kernel: parity of every variant first, then
# (a) bench.py config 2 / config 3 per-op rates, alternating, (b) every kernel at the
# gpubench hbm class.  TF_EW_V16: 0 = never, all = every op, unset = per-op default.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_variants.py -x -q -m gpu > gpurun_out/v16_tests.log 2>&1; echo rc=$? >> gpurun_out/v16_tests.log
o=gpurun_out/v16_ab.txt; : > $o
fmt='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print("value %.2f G  " % (d["value"]/1e9) + "  ".join("%s %.0f" % (k, v["gbs"]) for k, v in d["per_op"].items()) + "  sm_mhz %s" % d["clocks"]["sm_mhz"])'
for r in 1 2 3; do
  for v in 0 all; do
    export TF_EW_V16=$v
    echo -n "v16=$v c2  " >> $o
    timeout 600 python bench.py --no-sub-workloads --no-e2e --no-cpu-baseline --no-check --steps 20 --warmup 5 2>/dev/null | python -c "$fmt" >> $o
    echo -n "v16=$v c3  " >> $o
    timeout 600 python bench.py --workload config3 --no-e2e --no-cpu-baseline --no-check --steps 10 --warmup 3 2>/dev/null | python -c "$fmt" >> $o
  done
done
for r in 1 2; do
  for v in 0 all; do
    TF_EW_V16=$v timeout 900 python -m paper_1401_6235_b200.gpubench --sizes hbm --reps 7 > gpurun_out/v16_gpubench_${v}_$r.txt 2>&1
  done
done
unset TF_EW_V16
echo done >> $o
