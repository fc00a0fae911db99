"""Fused-kernel throughput vs composing the elementwise kernels (f64, n=2^27)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import kernels as K, fused as F, workloads as W


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


n = 1 << 27
ps = W.PlaneSet("config2", n, torch.float64, 0)
x0, x1, y0, y1 = ps.planes("vtadd2")
a = K.TwofoldArray(*ps.planes("vtsqrt1"))
X, Y = K.TwofoldArray(x0, x1), K.TwofoldArray(y0, y1)
t = K.empty_twofold(n, torch.float64)
o = K.empty_twofold(n, torch.float64)
res = {}
ms_f = timeit(lambda: F.vtaxpy(a, X, Y, o))
ms_c = timeit(lambda: (K.vtmul2(a, X, t), K.vtadd2(t, Y, o)))
res["axpy"] = {"fused_ms": ms_f, "composed_ms": ms_c, "fused_gbs": 64 * n / ms_f / 1e6,
               "speedup": ms_c / ms_f}
ms_f = timeit(lambda: F.vtsubmul(a, X, Y, o))
res["submul"] = {"fused_ms": ms_f, "fused_gbs": 64 * n / ms_f / 1e6}
q = tuple(K.empty_twofold(n, torch.float64) for _ in range(3))
cq = K.TwofoldArray(torch.abs(y0) * 1e-3, y1 * 1e-3)
ms = timeit(lambda: F.vtquadratic(a, X, cq, q))
res["quadratic"] = {"ms": ms, "G_inst_s": n / ms / 1e6, "gbs": 96 * n / ms / 1e6,
                    "inputs": "c = |y|*1e-3: about half the discriminants negative (NaN roots)"}
# real roots everywhere: c = b^2 / (4a) * U[0.1, 0.9] (disc > 0), tails at 2^-53 scale
g = torch.Generator(device="cuda").manual_seed(7)
u = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 0.8 + 0.1
c0 = x0 * x0 / (4 * a.value) * u
c1 = c0 * 2.0**-53 * (torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
cr = K.TwofoldArray(c0, c1)
ms = timeit(lambda: F.vtquadratic(a, X, cr, q))
res["quadratic_real_roots"] = {"ms": ms, "G_inst_s": n / ms / 1e6, "gbs": 96 * n / ms / 1e6,
                               "inputs": "c = b^2/(4a) * U[0.1, 0.9]: every discriminant positive"}
m = 1 << 24
Av = torch.rand((3, 3, m), dtype=torch.float64, device="cuda") + 4 * torch.eye(3, dtype=torch.float64, device="cuda")[:, :, None]
Ae = torch.zeros_like(Av)
fv = torch.rand((3, m), dtype=torch.float64, device="cuda")
fe = torch.zeros_like(fv)
xo = K.TwofoldArray(torch.empty_like(fv), torch.empty_like(fv))
ms = timeit(lambda: F.vtgauss3(K.TwofoldArray(Av, Ae), K.TwofoldArray(fv, fe), xo))
res["gauss3"] = {"ms": ms, "G_systems_s": m / ms / 1e6, "gbs": 240 * m / ms / 1e6}
print(json.dumps(res, indent=1))
