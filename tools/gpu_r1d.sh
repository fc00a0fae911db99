#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r1d
#timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu --durations=0 > ${o}_fullsize.log 2>&1; echo "rc=$?" >> ${o}_fullsize.log
export BENCH_DIST_BACKEND=gloo
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --elems 16777216 --steps 5 > ${o}_dry2_c2.json 2> ${o}_dry2_c2.err; echo "rc=$?" >> ${o}_dry2_c2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --workload config4 --elems 16777216 --steps 5 > ${o}_dry2_c4.json 2> ${o}_dry2_c4.err; echo "rc=$?" >> ${o}_dry2_c4.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --workload config5 --elems 4194304 --steps 5 > ${o}_dry2_c5.json 2> ${o}_dry2_c5.err; echo "rc=$?" >> ${o}_dry2_c5.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 2 --steps 2 > ${o}_dry2_ref.json 2> ${o}_dry2_ref.err; echo "rc=$?" >> ${o}_dry2_ref.err
echo done
