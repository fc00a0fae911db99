bash tools/gpu_suite.sh r1e tests smoke bench bench4 bench5 ref
timeout 300 python bench.py --impl reference --workload config4 --steps 3 > gpurun_out/r1e_ref4.json 2>&1
timeout 300 python bench.py --impl reference --workload config5 --steps 3 > gpurun_out/r1e_ref5.json 2>&1
nproc > gpurun_out/r1e_nproc.txt; lscpu | head -20 >> gpurun_out/r1e_nproc.txt
