# ncu --set full of every bench workload's kernels at the bench's exact shapes
# (tools/shape_launch.py; each command first runs clean without ncu), plus the
# launch list of the default bench command.  Outputs gpurun_out/ns_*.
mkdir -p gpurun_out
for c in ${NCU_CONFIGS:-config1 config2 config3 config4 config5}; do
  k='ew_(bulk_|step_|step16_)?kernel'; [ $c = config4 ] && k=reduce_kernel; [ $c = config5 ] && k=horner_kernel; [ $c = copy ] && k=dotted_vec_kernel
  cnt=$([ $c = config2 ] && echo 5 || ([ $c = config3 ] && echo 3 || ([ $c = copy ] && echo 1 || echo 2)))
  timeout 300 python tools/shape_launch.py $c --reps 1 > gpurun_out/ns_$c.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -c $cnt \
      -o gpurun_out/ns_$c python tools/shape_launch.py $c --reps 1 >> gpurun_out/ns_$c.log 2>&1
  echo "rc=$?" >> gpurun_out/ns_$c.log
done
