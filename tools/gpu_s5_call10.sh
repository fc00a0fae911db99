mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_elementwise.py -x -q -m gpu > gpurun_out/c10_ew_tests.log 2>&1; echo rc=$? >> gpurun_out/c10_ew_tests.log
: > gpurun_out/c10_half.jsonl
for v in default 0 default 0; do
  if [ $v = default ]; then unset TF_EW_V16; else export TF_EW_V16=0; fi
  timeout 300 python tools/halfaligned_probe.py >> gpurun_out/c10_half.jsonl 2>> gpurun_out/c10_half.err
done
