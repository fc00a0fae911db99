# e2e (host_batch over pinned planes, config 2) against the host pipeline's slots and chunk size
mkdir -p gpurun_out; o=gpurun_out/e2e_sweep2.txt; : > $o
fmt='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d["e2e"]
print("e2e %.3f G (frac %.3f, link duplex %.1f)  per_call %.3f G (frac %.3f)" % (e["value"]/1e9, e["roofline"]["frac"], e["roofline"]["link_gbs"]["duplex"], e["per_call"]["value"]/1e9, e["per_call"]["roofline"]["frac"]))'
for r in 1 2; do
for sl in 3 4 6; do for ch in 16 32 64; do
  echo -n "slots=$sl chunk=$ch  " >> $o
  TF_HOST_SLOTS=$sl TF_HOST_CHUNK_MB=$ch timeout 600 python bench.py --no-sub-workloads --no-cpu-baseline --no-check --no-device-batch --no-pageable --steps 3 --warmup 3 --e2e-steps 4 2>/dev/null | python -c "$fmt" >> $o
done; done; done
