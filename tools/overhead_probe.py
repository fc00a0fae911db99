"""Per-call host overhead of the Python drop-in (small n, device planes)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import kernels as K

n = 100
x = K.TwofoldArray(torch.rand(n, dtype=torch.float64, device="cuda"), torch.zeros(n, dtype=torch.float64, device="cuda"))
o = K.empty_twofold(n, torch.float64)
res = {}
for label, fn in (("validated vtadd2", lambda: K.vtadd2(x, x, o)),
                  ("raw loop", lambda: K.KERNELS["vtadd2"].loop(x.value, x.error, x.value, x.error, o.value, o.error))):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5000):
        fn()
    torch.cuda.synchronize()
    res[label] = (time.perf_counter() - t) / 5000 * 1e6
print(json.dumps({"us_per_call": res}))
