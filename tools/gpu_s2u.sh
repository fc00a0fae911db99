mkdir -p gpurun_out
timeout 600 python tools/fused_bench.py > gpurun_out/s2u_fused.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:quad_kernel -c 2 --csv --log-file gpurun_out/s2u_quad.csv python tools/fused_bench.py > gpurun_out/s2u_ncu.log 2>&1
