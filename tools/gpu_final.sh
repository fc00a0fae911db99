# Round-end style validation: the full GPU suite, smoke(), every bench workload,
# the reference arm, and the multi-rank dry runs.  Outputs: gpurun_out/fin_*.
mkdir -p gpurun_out
bash tools/gpu_suite.sh fin tests smoke bench bench1 bench3 bench4 bench5 ref
bash tools/gpu_multirank_dryrun.sh
