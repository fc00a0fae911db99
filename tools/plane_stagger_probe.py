"""Does the relative placement of the planes matter?  The six planes of a 22-arity op are views
into ONE buffer at offsets k * (plane + stagger): stagger = 0 puts every plane a whole 1 GiB
apart (what separate allocations give); other values shift plane k by k * stagger bytes.
f64, 2^27 elements, 20 launches back to back (events around the loop), default kernels."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import kernels as K

n = 1 << 27
res = {}
for stagger in (0, 256, 4096, 65536, (1 << 20) + 4096, 3 * (1 << 20) + 8192):
    se = stagger // 8
    buf = torch.rand(6 * (n + se) + 64, dtype=torch.float64, device="cuda") + 1
    pl = [buf[k * (n + se):k * (n + se) + n] for k in range(6)]
    row = {}
    for name, args in (("vtadd2", pl), ("vtdiv2", pl), ("vtsqrt1", pl[:2] + pl[4:])):
        f = K.KERNELS[name].loop
        for _ in range(3):
            f(*args)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            f(*args)
        b.record(); b.synchronize()
        row[name] = round(len(args) * n * 8 * 20 / (a.elapsed_time(b) * 1e-3) / 1e9)
    res[str(stagger)] = row
    del buf, pl
    torch.cuda.empty_cache()
print(json.dumps(res))
