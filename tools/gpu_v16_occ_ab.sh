# Resident CTAs per SM of the lean 16-byte kernel, capped by unused dynamic shared memory:
# vtdiv2 (48 registers, 5 CTAs/SM) streams 7.13 TB/s while vtadd2 (30 registers, 8 CTAs/SM)
# streams 7.02 over the same traffic — is lower residency better for the four-plane ops?
mkdir -p gpurun_out; : > gpurun_out/v16_occ.jsonl
for r in 1 2; do
  for sm in 0 32768 36864 45056; do
    echo -n "{\"smem\": $sm, \"run\": " >> gpurun_out/v16_occ.jsonl
    TF_EW_V16_SMEM=$sm timeout 600 python tools/ew_seq_ab.py >> gpurun_out/v16_occ.jsonl 2>> gpurun_out/v16_occ.err
    echo "}" >> gpurun_out/v16_occ.jsonl
  done
done
