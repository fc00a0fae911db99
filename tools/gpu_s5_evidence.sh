# Session-5 evidence for the final build: ncu --set full at every bench shape (incl. the
# vmem copy), summarised on the box (the reports themselves exceed the 64 MiB return
# limit and are deleted), then the ncu launch list of the default bench command (after it
# ran clean).
mkdir -p gpurun_out
for c in ${NCU_CONFIGS:-config2 copy config1 config3 config4 config5}; do
  NCU_CONFIGS=$c bash tools/gpu_ncu_shapes.sh
  if [ -f gpurun_out/ns_$c.ncu-rep ]; then
    python tools/ncu_summary.py gpurun_out/ns_$c.ncu-rep --json > gpurun_out/ns_$c.summary.json 2> gpurun_out/ns_$c.summary.err
    rm -f gpurun_out/ns_$c.ncu-rep
  fi
done
cmd="python bench.py --steps 2 --warmup 1"
timeout 900 $cmd > gpurun_out/s5_plain.json 2> gpurun_out/s5_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/s5_launches.csv $cmd > gpurun_out/s5_ncu_launches.log 2>&1
echo "rc=$?" >> gpurun_out/s5_ncu_launches.log
echo evidence-done
