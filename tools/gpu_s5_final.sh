# Session-5 validation of the final build on one fresh box: the GPU suite, smoke(), the
# default bench and the reference arm, then the ncu evidence (tools/gpu_s5_evidence.sh).
mkdir -p gpurun_out
bash tools/gpu_suite.sh s5f tests smoke bench ref
NCU_CONFIGS="config2 config1 config3" bash tools/gpu_s5_evidence.sh
timeout 900 python -m paper_1401_6235_b200.gpubench --sizes hbm --reps 7 > gpurun_out/s5f_gpubench_hbm.txt 2>&1
timeout 600 python tools/convert_bench.py > gpurun_out/s5f_convert.json 2> gpurun_out/s5f_convert.err
du -sh gpurun_out
