# (Record of a removed variant: TF_IL_LIGHT no longer exists in the library.)
# Interleaved layout: LIGHT lean kernel (TF_IL_LIGHT=all) vs the per-op defaults (TF_IL_LIGHT=0),
# all 22 ops launched one after another (tools/ew_seq_ab.py, SEQ_LAYOUT=interleaved).
mkdir -p gpurun_out; : > gpurun_out/il_light.jsonl
TF_IL_LIGHT=all timeout 900 python -m pytest tests/test_gpu_interleaved.py -x -q -m gpu > gpurun_out/il_light_tests.log 2>&1; echo rc=$? >> gpurun_out/il_light_tests.log
for r in 1 2 3; do for v in 0 all; do
  SEQ_LAYOUT=interleaved TF_IL_LIGHT=$v timeout 600 python tools/ew_seq_ab.py >> gpurun_out/il_light.jsonl 2>> gpurun_out/il_light.err
done; done
