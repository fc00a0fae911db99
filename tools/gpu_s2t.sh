mkdir -p gpurun_out
for w in config2 config3 config1; do
timeout 900 python bench.py --workload $w --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/s2t_$w.json 2> gpurun_out/s2t_$w.err; echo "rc=$?" >> gpurun_out/s2t_$w.err
done
