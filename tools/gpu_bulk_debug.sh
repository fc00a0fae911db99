mkdir -p gpurun_out
o=gpurun_out/bulk_debug.txt; : > $o
for v in main nst2_4 nst2_2; do
  for r in 8 4; do
    echo "## lib=$v reps=$r" >> $o
    if [ $v = main ]; then unset TF_LIB_PATH; else export TF_LIB_PATH=paper_1401_6235_b200/_lib/variants/$v/libtwofold_b200.so; fi
    TF_EW_BULK=all TF_EW_BULK_REPS=$r timeout 300 python tools/bulk_debug.py >> $o 2>&1
  done
done
unset TF_LIB_PATH
echo "## PDL off" >> $o
TF_PDL=0 TF_EW_BULK=all timeout 300 python tools/bulk_debug.py >> $o 2>&1
echo done >> $o
