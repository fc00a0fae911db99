# TMA-staged elementwise path (no scalar loops; head/tail in one extra CTA) vs the lean
# register kernel, per-op bench times on config 2 (f64 2^28) and config 3 (f32 2^30).
mkdir -p gpurun_out
TF_EW_BULK=all TF_EW_BULK_REPS=8 timeout 300 python tools/bulk_debug.py > gpurun_out/b2_debug.txt 2>&1
TF_EW_BULK=all TF_EW_BULK_REPS=2 timeout 600 python tools/sanitize_smoke.py > gpurun_out/b2_smoke.txt 2>&1; echo rc=$? >> gpurun_out/b2_smoke.txt
o=gpurun_out/b2_ab.txt; : > $o
for r in 1 2 3; do
  for v in lean bulk1 bulk2 bulk4; do
    case $v in lean) e="TF_EW_BULK=0";; bulk1) e="TF_EW_BULK=all TF_EW_BULK_REPS=1";; bulk2) e="TF_EW_BULK=all TF_EW_BULK_REPS=2";; bulk4) e="TF_EW_BULK=all TF_EW_BULK_REPS=4";; esac
    echo -n "$v " >> $o
    env $e timeout 600 python bench.py --no-sub-workloads --no-e2e --no-cpu-baseline --no-check --no-device-batch --steps 20 --warmup 5 2>/dev/null | tail -1 >> $o
    echo -n "$v-c3 " >> $o
    env $e timeout 600 python bench.py --workload config3 --no-e2e --no-cpu-baseline --no-check --no-device-batch --steps 10 --warmup 3 2>/dev/null | tail -1 >> $o
  done
done
echo done >> $o
