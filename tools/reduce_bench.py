"""Reduction and Horner throughput, f32 and f64 (CUDA-graph repeat loops)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import reduce as R, kernels as K, workloads as W
from paper_1401_6235_b200.gpubench import _measure, _peak_gbs

peak = _peak_gbs()
res = {}
for dt, name in ((torch.float64, "f64"), (torch.float32, "f32")):
    esz = 8 if dt == torch.float64 else 4
    n = (1 << 31) // esz  # 2 GiB per plane
    x = W.fill(torch.empty(n, dtype=dt, device="cuda"), W.UNIFORM, 1, 0, -1.0, 1.0)
    y = W.fill(torch.empty(n, dtype=dt, device="cuda"), W.UNIFORM, 2, 0, -1.0, 1.0)
    out = torch.empty(2, dtype=dt, device="cuda")
    for rop, fn, planes in (("vtsum", lambda: R.vtsum(x, out=out), 1),
                            ("vtsum2", lambda: R.vtsum2((x, y), out=out), 2),
                            ("vtdot", lambda: R.vtdot(x, y, out=out), 2)):
        fn()
        iters, best = _measure(fn, 5)
        t = best / iters
        gbs = planes * esz * n / t / 1e9
        res["%s_%s" % (rop, name)] = {"n": n, "ms": t * 1e3, "gbs": gbs, "frac_copy_peak": gbs / peak,
                                      "G_elem_s": n / t / 1e9}
    m = 1 << 26
    xs = W.fill(torch.empty(m, dtype=dt, device="cuda"), W.UNIFORM, 3, 0, 0.9, 1.1)
    o = K.empty_twofold(m, dt)
    c = R.binomial_coeffs(20)
    iters, best = _measure(lambda: R.vthorner(c, xs, o), 5)
    t = best / iters
    res["vthorner_%s" % name] = {"n": m, "ms": t * 1e3, "G_points_s": m / t / 1e9,
                                 "T_instr_s": 220 * m / t / 1e12}
print(json.dumps(res, indent=1))
