# Fused axpy / submul on 16-byte vs 32-byte vectors (TF_FUSED_VB=16), tools/fused_bench.py
mkdir -p gpurun_out; : > gpurun_out/fused_vb.txt
TF_FUSED_VB=16 timeout 600 python -m pytest tests/test_fused.py -x -q -m gpu > gpurun_out/fused_vb_tests.log 2>&1; echo rc=$? >> gpurun_out/fused_vb_tests.log
for r in 1 2 3; do for v in 32 16; do
  echo -n "vb=$v " >> gpurun_out/fused_vb.txt
  TF_FUSED_VB=$v timeout 600 python tools/fused_bench.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(' '.join('%s %.0f' % (k, v.get('fused_gbs', v.get('gbs', 0))) for k, v in d.items()))" >> gpurun_out/fused_vb.txt
done; done
