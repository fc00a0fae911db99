"""e2e host-path probe: pinned vs pageable numpy planes through kernels.vtadd2."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1401_6235_b200 import kernels as K

n = 1 << 27
res = {}
for kind in ("pinned", "pageable"):
    if kind == "pinned":
        x = [torch.rand(n, dtype=torch.float64).pin_memory().numpy() for _ in range(4)]
        out = K.empty_twofold(n, np.float64, device="cpu", pin_memory=True)
    else:
        x = [np.random.rand(n) for _ in range(4)]
        out = K.empty_twofold(n, np.float64, device="cpu")
        out.value[:] = 0; out.error[:] = 0
    X, Y = K.TwofoldArray(x[0], x[1]), K.TwofoldArray(x[2], x[3])
    import time as _t
    t1 = _t.perf_counter()
    K.vtadd2(X, Y, out)
    res[kind + "_first_call_s"] = _t.perf_counter() - t1
    for _ in range(K._REG_AFTER):  # pageable planes get page-locked on reuse
        K.vtadd2(X, Y, out)
    t = time.perf_counter()
    for _ in range(3):
        K.vtadd2(X, Y, out)
    dt = (time.perf_counter() - t) / 3
    res[kind] = {"melem_s": n / dt / 1e6, "gbs_moved": 48 * n / dt / 1e9}
print(json.dumps(res))
