# Final build of session 5: GPU suite (with durations), smoke(), both bench arms, fused bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu --durations=12 > gpurun_out/s5g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5g_pytest.log
bash tools/gpu_suite.sh s5g smoke bench ref
timeout 600 python tools/fused_bench.py > gpurun_out/s5g_fused.json 2>&1
