#!/bin/bash
mkdir -p gpurun_out
for slots in 3 4 6; do for mb in 16 32 64; do
  TF_HOST_SLOTS=$slots TF_HOST_CHUNK_MB=$mb timeout 300 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/sw_${slots}_${mb}.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw_${slots}_${mb}.json')); e=d['e2e']; print($slots, $mb, round(e['value']/1e9,3), round(e['batched']['value']/1e9,3), round(e['roofline']['frac'],3))" >> gpurun_out/e2e_sweep.txt
done; done
