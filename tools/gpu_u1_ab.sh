# One-plane ops (vtsqrt) on the 32-byte lean kernel: vectors in flight per thread 2 (default) / 1 / 4
# (library variants -DTF_U_NIN1), all 22 ops launched one after another (tools/ew_seq_ab.py).
mkdir -p gpurun_out; : > gpurun_out/u1_ab.jsonl
V=$PWD/paper_1401_6235_b200/_lib/variants
for r in 1 2 3; do for v in base u1 u4; do
  unset TF_LIB_PATH; [ $v != base ] && export TF_LIB_PATH=$V/$v/libtwofold_b200.so
  echo -n "{\"variant\": \"$v\", \"run\": " >> gpurun_out/u1_ab.jsonl
  timeout 600 python tools/ew_seq_ab.py >> gpurun_out/u1_ab.jsonl 2>> gpurun_out/u1_ab.err
done; done
