# Round-end style validation: the full GPU suite, smoke(), every bench workload,
# the reference arm, the multi-rank dry runs, the all-kernel gpubench table and
# the fused-kernel bench.  Outputs: gpurun_out/fin_*, mr_*.
mkdir -p gpurun_out
bash tools/gpu_suite.sh fin tests smoke bench bench1 bench3 bench4 bench5 ref
bash tools/gpu_multirank_dryrun.sh
timeout 1500 python -m paper_1401_6235_b200.gpubench --csv gpurun_out/fin_gpubench.csv > gpurun_out/fin_gpubench.txt 2>&1
timeout 600 python tools/fused_bench.py > gpurun_out/fin_fused.json 2>&1
