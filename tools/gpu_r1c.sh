#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r1c
timeout 120 python tools/pcie_probe.py > ${o}_pcie.json 2>&1
for slots in 3 4; do for mb in 16 64; do
  TF_HOST_SLOTS=$slots TF_HOST_CHUNK_MB=$mb timeout 120 python tools/pcie_probe.py e2e >> ${o}_e2e_sweep.json 2>&1
done; done
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $cmd > ${o}_plain_ew.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ew_kernel -s 5 -c 5 -o ${o}_prof_ew $cmd > ${o}_ncu_ew.log 2>&1; echo "rc=$?" >> ${o}_ncu_ew.log
cmd="python bench.py --workload config4 --steps 2 --warmup 1"
timeout 300 $cmd > ${o}_plain_red.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:reduce_kernel -c 2 -o ${o}_prof_red $cmd > ${o}_ncu_red.log 2>&1; echo "rc=$?" >> ${o}_ncu_red.log
cmd="python bench.py --workload config5 --steps 2 --warmup 1"
timeout 300 $cmd > ${o}_plain_h.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:horner -c 1 -o ${o}_prof_horner $cmd > ${o}_ncu_h.log 2>&1; echo "rc=$?" >> ${o}_ncu_h.log
echo done
