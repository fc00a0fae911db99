"""vthorner (x-1)^20 throughput, f64 and f32, 2^26 points, CUDA-event timed."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import kernels as K, reduce as R

res = {}
for dt in (torch.float64, torch.float32):
    n = 1 << 26
    x = torch.rand(n, dtype=dt, device="cuda") * 0.2 + 0.9
    out = K.empty_twofold(n, dt)
    c = R.binomial_coeffs(20)
    for _ in range(3):
        R.vthorner(c, x, out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        R.vthorner(c, x, out)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 20
    res[str(dt)] = {"G_points_s": n / ms / 1e6, "T_instr_s": 220 * n / ms / 1e9}
print(json.dumps(res))
