mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_elementwise.py -x -q -m gpu -k "batch" > gpurun_out/s2d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s2d_pytest.log
timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/s2d_bench.json 2> gpurun_out/s2d_bench.err; echo "rc=$?" >> gpurun_out/s2d_bench.err
timeout 600 python bench.py --workload config3 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/s2d_bench3.json 2> gpurun_out/s2d_bench3.err; echo "rc=$?" >> gpurun_out/s2d_bench3.err
timeout 600 python bench.py --workload config1 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/s2d_bench1.json 2> gpurun_out/s2d_bench1.err; echo "rc=$?" >> gpurun_out/s2d_bench1.err
