mkdir -p gpurun_out
for m in write write-read write write-read; do
timeout 300 python bench.py --workload config1 --steps 50 --l2-flush $m --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$m', round(d['value']/1e9,2), round(d['roofline']['frac'],3), d['ms_per_step'], {k:(round(v['ms']*1e3,2), round(v['gbs'])) for k,v in d['per_op'].items()})
" >> gpurun_out/s2c_flush.txt
done
