# every kernel at the gpubench hbm class: lean register path vs TMA-staged with 2 tiles per CTA
mkdir -p gpurun_out
for r in 1 2; do
  TF_EW_BULK=0 timeout 900 python -m paper_1401_6235_b200.gpubench --sizes hbm --reps 7 > gpurun_out/b3_lean_$r.txt 2>&1
  TF_EW_BULK=all TF_EW_BULK_REPS=2 timeout 900 python -m paper_1401_6235_b200.gpubench --sizes hbm --reps 7 > gpurun_out/b3_bulk2_$r.txt 2>&1
done
# interleaved layout: lean step kernel (default) vs ew_il_kernel
timeout 1200 python -m pytest tests/test_gpu_interleaved.py -x -q -m gpu > gpurun_out/il_tests.log 2>&1; echo rc=$? >> gpurun_out/il_tests.log
TF_IL_LEAN=0 timeout 1200 python -m pytest tests/test_gpu_interleaved.py -x -q -m gpu > gpurun_out/il_tests_old.log 2>&1; echo rc=$? >> gpurun_out/il_tests_old.log
for r in 1 2; do
  timeout 900 python -m paper_1401_6235_b200.gpubench --sizes hbm --reps 7 --layout interleaved > gpurun_out/b3_il_lean_$r.txt 2>&1
  TF_IL_LEAN=0 timeout 900 python -m paper_1401_6235_b200.gpubench --sizes hbm --reps 7 --layout interleaved > gpurun_out/b3_il_old_$r.txt 2>&1
done
