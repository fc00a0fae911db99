#!/bin/bash
# A/B of the TMA-staged elementwise variant (ew_bulk_kernel) against the register
# path on the config-2 planes (n = 2^28, f64) and config-3 planes (2^30, f32).
# Output: gpurun_out/bulk_ab.txt
mkdir -p gpurun_out
o=gpurun_out/bulk_ab.txt
: > $o
ops=vtsqrt1,vtadd2,vtsub2,vtmul2,vtdiv2
for round in 1 2; do
  echo "## round $round" >> $o
  for v in reg bulk_r4 bulk_r8 bulk_r16 nst2_4 nst2_2; do
    case $v in
      reg)      env="TF_EW_BULK=0" ; lib="" ;;
      bulk_r4)  env="TF_EW_BULK=all TF_EW_BULK_REPS=4" ; lib="" ;;
      bulk_r8)  env="TF_EW_BULK=all TF_EW_BULK_REPS=8" ; lib="" ;;
      bulk_r16) env="TF_EW_BULK=all TF_EW_BULK_REPS=16" ; lib="" ;;
      nst2_4)   env="TF_EW_BULK=all" ; lib="paper_1401_6235_b200/_lib/variants/nst2_4/libtwofold_b200.so" ;;
      nst2_2)   env="TF_EW_BULK=all" ; lib="paper_1401_6235_b200/_lib/variants/nst2_2/libtwofold_b200.so" ;;
    esac
    echo -n "$v " >> $o
    if [ -n "$lib" ]; then export TF_LIB_PATH=$lib; else unset TF_LIB_PATH; fi
    env $env timeout 300 python tools/ew_ab.py --ops $ops --reps 40 >> $o 2>&1
  done
done
unset TF_LIB_PATH
echo "## config3 f32 (2^30)" >> $o
for v in reg bulk_r8; do
  case $v in reg) env="TF_EW_BULK=0";; bulk_r8) env="TF_EW_BULK=all TF_EW_BULK_REPS=8";; esac
  echo -n "$v " >> $o
  env $env timeout 300 python tools/ew_ab.py --config config3 --n 1073741824 --ops vtadd2,vtmul2,vtdiv2 --reps 20 >> $o 2>&1
done
echo done >> $o
