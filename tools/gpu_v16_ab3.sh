mkdir -p gpurun_out; : > gpurun_out/v16_seq.jsonl
for r in 1 2 3; do for v in 0 all; do TF_EW_V16=$v timeout 600 python tools/ew_seq_ab.py >> gpurun_out/v16_seq.jsonl 2>> gpurun_out/v16_seq.err; done; done
