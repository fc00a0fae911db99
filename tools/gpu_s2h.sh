mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_variants.py tests/test_gpu_reduce.py tests/test_c_abi.py -x -q -m gpu > gpurun_out/s2h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s2h_pytest.log
timeout 600 python bench.py --workload config1 --steps 30 --no-cpu-baseline > gpurun_out/s2h_bench1.json 2> gpurun_out/s2h_bench1.err
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-device-batch > gpurun_out/s2h_bench.json 2> gpurun_out/s2h_bench.err
