# Round-2 session-3 validation + evidence: full GPU suite, smoke, fused bench,
# ncu --set full of the config-2 kernels and the vmem copy at 2^28, the launch
# list of the default bench, the default bench line and the reference arm.
mkdir -p gpurun_out
bash tools/gpu_suite.sh s3f tests smoke
timeout 600 python tools/fused_bench.py > gpurun_out/s3f_fused.json 2>&1
NCU_CONFIGS="config2 copy" bash tools/gpu_ncu_shapes.sh
cmd="python bench.py --steps 2 --warmup 1"
timeout 900 $cmd > gpurun_out/s3f_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/s3f_launches.csv $cmd > gpurun_out/s3f_ncu_launches.log 2>&1; echo "rc=$?" >> gpurun_out/s3f_ncu_launches.log
bash tools/gpu_suite.sh s3f bench ref
