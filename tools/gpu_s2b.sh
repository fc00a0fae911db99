mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_reduce.py -x -q -m gpu -k "p2p or xgpu or sharded" > gpurun_out/s2b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s2b_pytest.log
timeout 600 python bench.py --steps 10 > gpurun_out/s2b_bench.json 2> gpurun_out/s2b_bench.err; echo "rc=$?" >> gpurun_out/s2b_bench.err
timeout 600 python bench.py --workload config4 --steps 10 > gpurun_out/s2b_bench4.json 2> gpurun_out/s2b_bench4.err; echo "rc=$?" >> gpurun_out/s2b_bench4.err
