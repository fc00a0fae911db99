# (Record of a removed variant: TF_BATCH_PREFETCH no longer exists in the library.)
# Device batch: L2 prefetch of the later ops' first-read planes (default) vs none
# (TF_BATCH_PREFETCH=0).  Parity first, then alternating bench runs on one box.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_large_index.py tests/test_gpu_variants.py -x -q -m gpu -k "batch or variant" > gpurun_out/pf_tests.log 2>&1; echo rc=$? >> gpurun_out/pf_tests.log
o=gpurun_out/batch_pf_ab.txt; : > $o
fmt='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=d["device_batch"]
print("device_batch %.1f G elem-ops/s (%.0f GB/s, %.4f ms/step)  value %.2f G  sm_mhz %s" % (b["value"]/1e9, b["roofline"]["achieved"], b["ms_per_step"], d["value"]/1e9, d["clocks"]["sm_mhz"]))'
for r in 1 2 3; do
  for v in pf nopf; do
    if [ $v = pf ]; then unset TF_BATCH_PREFETCH; else export TF_BATCH_PREFETCH=0; fi
    echo -n "$v      " >> $o
    timeout 600 python bench.py --no-sub-workloads --no-e2e --no-cpu-baseline --no-check --steps 20 --warmup 5 2>/dev/null | python -c "$fmt" >> $o
    echo -n "$v-c3   " >> $o
    timeout 600 python bench.py --workload config3 --no-e2e --no-cpu-baseline --no-check --steps 10 --warmup 3 2>/dev/null | python -c "$fmt" >> $o
    echo -n "$v-c1   " >> $o
    timeout 600 python bench.py --workload config1 --no-e2e --no-cpu-baseline --no-check --steps 50 --warmup 5 2>/dev/null | python -c "$fmt" >> $o
  done
done
unset TF_BATCH_PREFETCH
echo done >> $o
