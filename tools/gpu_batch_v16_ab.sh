# Device batch: lean 16-byte kernel (TF_BATCH_V16=1; register caps 6/5/4 CTAs per SM as
# library variants) vs the default (lean 32-byte for f64, batch_kernel for f32).
mkdir -p gpurun_out
TF_BATCH_V16=1 timeout 900 python tools/sanitize_smoke.py > gpurun_out/bv16_smoke.log 2>&1; echo rc=$? >> gpurun_out/bv16_smoke.log
TF_BATCH_V16=1 timeout 900 python -m pytest tests/test_gpu_elementwise.py -x -q -m gpu -k batch > gpurun_out/bv16_tests.log 2>&1; echo rc=$? >> gpurun_out/bv16_tests.log
o=gpurun_out/batch_v16_ab.txt; : > $o
fmt='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=d["device_batch"]
print("device_batch %.1f G elem-ops/s (%.0f GB/s, %.4f ms/step)  value %.2f G  sm_mhz %s" % (b["value"]/1e9, b["roofline"]["achieved"], b["ms_per_step"], d["value"]/1e9, d["clocks"]["sm_mhz"]))'
V=paper_1401_6235_b200/_lib/variants
for r in 1 2 3; do
  for v in base v16m6 v16m5 v16m4; do
    unset TF_BATCH_V16 TF_LIB_PATH
    case $v in
      v16m6) export TF_BATCH_V16=1;;
      v16m5) export TF_BATCH_V16=1 TF_LIB_PATH=$PWD/$V/b5/libtwofold_b200.so;;
      v16m4) export TF_BATCH_V16=1 TF_LIB_PATH=$PWD/$V/b4/libtwofold_b200.so;;
    esac
    echo -n "$v c2  " >> $o
    timeout 600 python bench.py --no-sub-workloads --no-e2e --no-cpu-baseline --no-check --steps 20 --warmup 5 2>/dev/null | python -c "$fmt" >> $o
    echo -n "$v c3  " >> $o
    timeout 600 python bench.py --workload config3 --no-e2e --no-cpu-baseline --no-check --steps 10 --warmup 3 2>/dev/null | python -c "$fmt" >> $o
    echo -n "$v c1  " >> $o
    timeout 600 python bench.py --workload config1 --no-e2e --no-cpu-baseline --no-check --steps 50 --warmup 5 2>/dev/null | python -c "$fmt" >> $o
  done
done
unset TF_BATCH_V16 TF_LIB_PATH
echo done >> $o
