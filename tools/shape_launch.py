"""Launch the bench's dominant kernels at exactly the bench's shapes, a few
times each, for ncu captures (`ncu --set full -k regex:... python
tools/shape_launch.py config2`).  Inputs are the bench's own (workloads.py).

    python tools/shape_launch.py config1|config2|config3|config4|config5|copy [--reps 2]

`copy`: the vmem baseline (tf_dotted base 4, f64, 2^28) - a 1:1 read/write
stream like vtsqrt1, for comparing DRAM efficiency at the same traffic mix.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1401_6235_b200 import kernels as K, reduce as R, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
OPS = {"config1": ["vtadd2", "vtmul2"], "config2": ["vtadd2", "vtsub2", "vtmul2", "vtdiv2", "vtsqrt1"],
       "config3": ["vtadd2", "vtmul2", "vtdiv2"]}
N = {"config1": 1 << 20, "config2": 1 << 28, "config3": 1 << 30, "config4": 1 << 30,
     "config5": 1 << 26, "copy": 1 << 28}
n = N[a.config]
if a.config in OPS:
    dt = torch.float32 if a.config == "config3" else torch.float64
    ps = W.PlaneSet(a.config, n, dt, 0)
    out = K.empty_twofold(n, dt)
    for name in OPS[a.config]:
        planes = ps.planes(name)
        for _ in range(a.reps):
            K.KERNELS[name].loop(*planes, out.value, out.error)
elif a.config == "copy":
    from paper_1401_6235_b200 import _lib

    n = 1 << 28
    x = W.fill(torch.empty(n, dtype=torch.float64, device="cuda"), W.UNIFORM, 1, 0, -1.0, 1.0)
    r = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(a.reps):
        _lib.check(_lib.lib().tf_dotted(4, _lib.TF_F64, n, x.data_ptr(), None, r.data_ptr(), s),
                   "tf_dotted")
elif a.config == "config4":
    X, Y, P = W.config4_planes(n, 0, n, "cuda")
    o = torch.empty(2, dtype=torch.float64, device="cuda")
    for _ in range(a.reps):
        R.vtdot(X, Y, out=o)
    for _ in range(a.reps):
        R.vtsum(P, out=o)
else:
    x = W.fill(torch.empty(n, dtype=torch.float64, device="cuda"), W.UNIFORM, 555, 0, 0.9, 1.1)
    out = K.empty_twofold(n, torch.float64)
    c = R.binomial_coeffs(20)
    for _ in range(a.reps):
        R.vthorner(c, x, out)
torch.cuda.synchronize()
print("ok", a.config, n)
