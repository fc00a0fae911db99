mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_elementwise.py tests/test_c_abi.py -x -q -m gpu > gpurun_out/s2x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s2x_pytest.log
TF_HOST_ZEROCOPY_MB=0 timeout 600 python tools/zerocopy_probe.py > gpurun_out/s2x_zc.json 2>&1
timeout 600 python tools/small_host_probe.py > gpurun_out/s2x_small.json 2>&1
timeout 600 python bench.py --workload config1 --steps 30 --no-cpu-baseline > gpurun_out/s2x_bench1.json 2> gpurun_out/s2x_bench1.err
