# lean batch kernel (batch_step_kernel, default) vs batch_kernel (TF_BATCH_LEAN=0)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_large_index.py tests/test_gpu_variants.py -x -q -m gpu -k "batch or variant" > gpurun_out/batch_tests.log 2>&1; echo rc=$? >> gpurun_out/batch_tests.log
o=gpurun_out/batch_ab.txt; : > $o
for r in 1 2 3; do
  for v in lean old; do
    if [ $v = lean ]; then unset TF_BATCH_LEAN; else export TF_BATCH_LEAN=0; fi
    echo -n "$v " >> $o
    timeout 600 python bench.py --no-sub-workloads --no-e2e --no-cpu-baseline --no-check --steps 20 --warmup 5 2>/dev/null | tail -1 >> $o
    echo -n "$v-c3 " >> $o
    timeout 600 python bench.py --workload config3 --no-e2e --no-cpu-baseline --no-check --steps 10 --warmup 3 2>/dev/null | tail -1 >> $o
    echo -n "$v-c1 " >> $o
    timeout 600 python bench.py --workload config1 --no-e2e --no-cpu-baseline --no-check --steps 50 --warmup 5 2>/dev/null | tail -1 >> $o
  done
done
unset TF_BATCH_LEAN
echo done >> $o
