mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_elementwise.py -x -q -m gpu > gpurun_out/s2e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s2e_pytest.log
