# Multi-rank code paths of bench.py on ONE GPU (no kernel waits on another rank):
# torchrun with NCCL at world 1; gloo dry runs at world 2 and 4 (every rank on
# cuda:0, partials exchanged through host tensors) in both scaling modes, with
# the default run's sub-workloads (config 4's bits asserted equal to N = 1);
# the reference arm under torchrun.  Small sizes (2^24 per rank / in total).
# Outputs: gpurun_out/mr_*.
mkdir -p gpurun_out
o=gpurun_out/mr
E="--elems 16777216 --sub-elems 16777216 --steps 5 --warmup 3 --e2e-steps 1 --cpu-sample 1048576"
run() { tag=$1; shift; timeout 900 "$@" > ${o}_$tag.json 2> ${o}_$tag.err; echo "rc=$?" >> ${o}_$tag.err; }
run tr1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 $E
for w in 2 4; do
  for sc in weak strong; do
    BENCH_DIST_BACKEND=gloo run tr${w}_$sc python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $((29520 + w * 2 + ${#sc})) bench.py --gpus $w --scaling $sc $E
  done
done
run tr2ref python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --ref-elems 1048576
