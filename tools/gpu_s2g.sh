mkdir -p gpurun_out
cmd="python bench.py --workload config1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --graph off"
timeout 300 $cmd > gpurun_out/s2g_plain.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max --clock-control none -k regex:"ew_kernel|batch_kernel" --csv \
   --log-file gpurun_out/s2g_launches.csv $cmd > gpurun_out/s2g_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/s2g_ncu.log
