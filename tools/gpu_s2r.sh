mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_fullsize.py -x -q -m gpu -k "ill or config4" > gpurun_out/s2r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s2r_pytest.log
timeout 900 python bench.py --workload config4 --steps 20 > gpurun_out/s2r_bench4.json 2> gpurun_out/s2r_bench4.err; echo "rc=$?" >> gpurun_out/s2r_bench4.err
