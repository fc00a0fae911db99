# all f64 kernels at the gpubench hbm class: register path vs TMA-staged path, then the default bench
mkdir -p gpurun_out
for r in 1 2; do
TF_EW_BULK=0 timeout 900 python -m paper_1401_6235_b200.gpubench --format f64 --sizes hbm --reps 7 > gpurun_out/gb_reg_$r.txt 2>&1
TF_EW_BULK=all timeout 900 python -m paper_1401_6235_b200.gpubench --format f64 --sizes hbm --reps 7 > gpurun_out/gb_bulk_$r.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo rc=$? >> gpurun_out/s5_bench.err
