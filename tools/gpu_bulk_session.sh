mkdir -p gpurun_out
bash tools/gpu_bulk_debug.sh
TF_EW_BULK=all timeout 900 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_large_index.py tests/test_gpu_fullsize.py tests/test_gpu_reduce.py -x -q -m gpu > gpurun_out/bulk_tests_all.log 2>&1; echo rc=$? >> gpurun_out/bulk_tests_all.log
bash tools/gpu_bulk_ab.sh
