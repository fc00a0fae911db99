# full GPU suite + benches + ncu of the device-batch kernel (round 1, session 2)
mkdir -p gpurun_out
bash tools/gpu_suite.sh s2f tests smoke bench bench1 bench3 bench4 bench5 ref
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:batch_kernel --csv \
   --log-file gpurun_out/s2f_batch_launches.csv $cmd > gpurun_out/s2f_ncu_batch.log 2>&1; echo "rc=$?" >> gpurun_out/s2f_ncu_batch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -c 1 \
   -o gpurun_out/s2f_prof_batch $cmd > gpurun_out/s2f_ncu_batch_full.log 2>&1; echo "rc=$?" >> gpurun_out/s2f_ncu_batch_full.log
