# Launch-bounds A/B (min resident CTAs): main build vs div2_mb4 (vtdiv2 at <= 64 registers)
# vs mb4all (every 32-byte-vector kernel and the batch kernel at <= 64).  Config-2 bench
# per-op times and the device batch, alternating builds; then gpubench f64 hbm.
mkdir -p gpurun_out
o=gpurun_out/minb_ab.txt; : > $o
for r in 1 2 3; do
  for v in main div2_mb4 mb4all; do
    if [ $v = main ]; then unset TF_LIB_PATH; else export TF_LIB_PATH=paper_1401_6235_b200/_lib/variants/$v/libtwofold_b200.so; fi
    echo -n "$v " >> $o
    timeout 600 python bench.py --no-sub-workloads --no-e2e --no-cpu-baseline --no-check --steps 20 --warmup 5 2>/dev/null | tail -1 >> $o
  done
done
for v in main mb4all; do
  if [ $v = main ]; then unset TF_LIB_PATH; else export TF_LIB_PATH=paper_1401_6235_b200/_lib/variants/$v/libtwofold_b200.so; fi
  timeout 900 python -m paper_1401_6235_b200.gpubench --format f64 --sizes hbm --reps 7 > gpurun_out/minb_gb_$v.txt 2>&1
done
unset TF_LIB_PATH
echo done >> $o
