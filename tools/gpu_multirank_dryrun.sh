# Multi-rank code paths of bench.py on ONE GPU (no kernel waits on another rank):
# torchrun with NCCL at world 1, gloo dry runs at world 2 (both ranks on cuda:0),
# and the reference arm under torchrun.  Outputs: gpurun_out/mr_*.
mkdir -p gpurun_out
o=gpurun_out/mr
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --elems 16777216 > ${o}_tr1.json 2> ${o}_tr1.err; echo "rc=$?" >> ${o}_tr1.err
BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 --elems 16777216 > ${o}_tr2.json 2> ${o}_tr2.err; echo "rc=$?" >> ${o}_tr2.err
BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --workload config4 --steps 5 --warmup 3 --elems 16777216 > ${o}_tr2c4.json 2> ${o}_tr2c4.err; echo "rc=$?" >> ${o}_tr2c4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > ${o}_tr2ref.json 2> ${o}_tr2ref.err; echo "rc=$?" >> ${o}_tr2ref.err
