#!/bin/bash
# Round-1 refresh: full GPU suite + all bench workloads + reference arms + launch list
bash tools/gpu_suite.sh r1i tests smoke bench bench1 bench3 bench4 bench5 ref launches
timeout 300 python bench.py --impl reference --workload config4 --steps 3 > gpurun_out/r1i_ref4.json 2>&1
timeout 300 python bench.py --impl reference --workload config5 --steps 3 > gpurun_out/r1i_ref5.json 2>&1
