"""Why does the in-process cpu_baseline leg run slower than the reference arm's
fresh process?  Times the oracle's Horner and dot (all host threads) at stages of
one process: before CUDA, after torch CUDA init, after device kernels, after the
host pipeline (pinned), after pageable host calls (page-locking), after
release_memory().  One JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as o  # noqa: E402

nt = os.cpu_count()
c = [float((-1) ** (20 - k) * __import__("math").comb(20, k)) for k in range(21)]
xs = np.random.default_rng(1).uniform(0.9, 1.1, 1 << 24)
oo = (np.zeros_like(xs), np.zeros_like(xs))
a = np.random.default_rng(2).uniform(-1, 1, 1 << 26)
b = np.random.default_rng(3).uniform(-1, 1, 1 << 26)
res = {"threads": nt}


def t(tag):
    def best(fn):
        fn()
        r = []
        for _ in range(3):
            t0 = time.perf_counter()
            fn()
            r.append(time.perf_counter() - t0)
        return min(r)
    res[tag] = {"horner_Gpts": xs.size / best(lambda: o.horner(c, xs, nthreads=nt, out=oo)) / 1e9,
                "dot_Gelem": a.size / best(lambda: o.reduce("dot", a, b, nthreads=nt)) / 1e9}


t("fresh")
import torch  # noqa: E402

torch.cuda.init()
torch.zeros(1, device="cuda")
t("after_cuda_init")
from paper_1401_6235_b200 import kernels as K, reduce as R  # noqa: E402

X = torch.from_numpy(a).cuda()
Y = torch.from_numpy(b).cuda()
for _ in range(20):
    R.vtdot(X, Y)
torch.cuda.synchronize()
t("after_device_kernels")
xh = torch.empty(1 << 26, dtype=torch.float64, pin_memory=True).numpy()
xh[:] = a
for _ in range(3):
    R.vtdot(xh, xh)
t("after_host_pipeline_pinned")
ap = a.copy()
for _ in range(6):
    R.vtdot(ap, ap)
t("after_pageable_calls")
res["torch_threads"] = torch.get_num_threads()
print(json.dumps(res), flush=True)
