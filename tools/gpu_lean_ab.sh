# lean single-step elementwise kernel (default) vs the chunked ew_kernel (TF_EW_LEAN=0):
# parity first, then the config-2/3 bench per-op times alternating, then gpubench hbm.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_variants.py tests/test_gpu_fullsize.py tests/test_gpu_large_index.py tests/test_gpu_interleaved.py tests/test_gpu_fast_ieee.py -x -q -m gpu > gpurun_out/lean_tests.log 2>&1; echo rc=$? >> gpurun_out/lean_tests.log
o=gpurun_out/lean_ab.txt; : > $o
for r in 1 2 3; do
  for v in lean chunked; do
    if [ $v = lean ]; then unset TF_EW_LEAN; else export TF_EW_LEAN=0; fi
    echo -n "$v " >> $o
    timeout 600 python bench.py --no-sub-workloads --no-e2e --no-cpu-baseline --no-check --steps 20 --warmup 5 2>/dev/null | tail -1 >> $o
    echo -n "$v-c3 " >> $o
    timeout 600 python bench.py --workload config3 --no-e2e --no-cpu-baseline --no-check --no-device-batch --steps 10 --warmup 3 2>/dev/null | tail -1 >> $o
  done
done
unset TF_EW_LEAN
for v in lean chunked; do
  if [ $v = lean ]; then unset TF_EW_LEAN; else export TF_EW_LEAN=0; fi
  timeout 900 python -m paper_1401_6235_b200.gpubench --sizes hbm,large --reps 7 > gpurun_out/lean_gb_$v.txt 2>&1
done
unset TF_EW_LEAN
echo done >> $o
