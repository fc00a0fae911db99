#!/bin/bash
# Build an A/B variant of libtwofold_b200.so with extra nvcc defines:
#   tools/build_variant.sh NAME "-DFOO=1 -DBAR"
# -> paper_1401_6235_b200/_lib/variants/NAME/libtwofold_b200.so (load with TF_LIB_PATH)
set -e
cd "$(dirname "$0")/../paper_1401_6235_b200/csrc"
name=$1; shift
out=../_lib/variants/$name
mkdir -p $out/obj
NV="/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -std=c++17 -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-ffp-contract=off"
for f in elementwise batch interleaved fused reduce horner hostpipe xgpu runtime gen_ill; do
  $NV "$@" -c $f.cu -o $out/obj/$f.o &
done
g++ -O3 -fPIC -std=c++17 -ffp-contract=off -c gen_dot.cpp -o $out/obj/gen_dot.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libtwofold_b200.so $out/obj/*.o -lpthread
echo built $out/libtwofold_b200.so
