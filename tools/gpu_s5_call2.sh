mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_interleaved.py -x -q -m gpu > gpurun_out/c2_il_tests.log 2>&1; echo rc=$? >> gpurun_out/c2_il_tests.log
for v in 1 0 1 0; do TF_CONV_LEAN=$v timeout 300 python tools/convert_bench.py >> gpurun_out/c2_convert.jsonl 2>> gpurun_out/c2_convert.err; done
bash tools/gpu_batch_pf_ab.sh
bash tools/gpu_s5_evidence.sh
du -sh gpurun_out
