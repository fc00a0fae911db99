# ncu --set full of the session-2 kernels: the reduction pair (config 4), an
# interleaved kernel and the fused axpy, each after its command ran clean without ncu.
mkdir -p gpurun_out
c4="python bench.py --workload config4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $c4 > gpurun_out/nx_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reduce_pair_kernel -c 1 \
  -o gpurun_out/nx_pair $c4 > gpurun_out/nx_pair.log 2>&1; echo "rc=$?" >> gpurun_out/nx_pair.log
il="python -m paper_1401_6235_b200.gpubench --sizes hbm --layout interleaved --ops vtadd2,vtmul1 --format f64 --reps 3"
timeout 600 $il > gpurun_out/nx_il.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:ew_il_kernel -c 2 -o gpurun_out/nx_il $il > gpurun_out/nx_il_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/nx_il_ncu.log
fb="python tools/fused_bench.py"
timeout 600 $fb > gpurun_out/nx_fb.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:fused_ew_kernel -c 2 -o gpurun_out/nx_fused $fb > gpurun_out/nx_fused_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/nx_fused_ncu.log
