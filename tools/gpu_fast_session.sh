# fast-path + TMA-staged variants: correctness first, then the A/B at the gpubench hbm class
mkdir -p gpurun_out
TF_EW_BULK=all TF_EW_BULK_REPS=8 timeout 300 python tools/bulk_debug.py > gpurun_out/f2_bulk_debug.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fast_ieee.py tests/test_gpu_elementwise.py tests/test_gpu_fullsize.py tests/test_gpu_variants.py tests/test_gpu_interleaved.py -x -q -m gpu > gpurun_out/f2_tests.log 2>&1; echo rc=$? >> gpurun_out/f2_tests.log
OPS=vtdiv2,vtdiv1,vtdiv,vtsqrt1,vtsqrt,vpdiv2,vpdiv1,vtadd2
for r in 1 2; do
TF_EW_BULK=0 timeout 900 python -m paper_1401_6235_b200.gpubench --format f64 --sizes hbm --reps 7 --ops $OPS > gpurun_out/f2gb_reg_$r.txt 2>&1
TF_EW_BULK=all timeout 900 python -m paper_1401_6235_b200.gpubench --format f64 --sizes hbm --reps 7 --ops $OPS > gpurun_out/f2gb_bulk_$r.txt 2>&1
for v in nst2_4 nst2_2; do
TF_LIB_PATH=paper_1401_6235_b200/_lib/variants/$v/libtwofold_b200.so TF_EW_BULK=all timeout 600 python -m paper_1401_6235_b200.gpubench --format f64 --sizes hbm --reps 7 --ops $OPS > gpurun_out/f2gb_${v}_$r.txt 2>&1
done
done
timeout 900 python -m paper_1401_6235_b200.gpubench --format f64 --sizes hbm --reps 7 --layout interleaved > gpurun_out/f2gb_il.txt 2>&1
timeout 900 python bench.py --no-sub-workloads > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo rc=$? >> gpurun_out/f2_bench.err
