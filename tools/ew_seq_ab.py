"""Every registry kernel in bench.py's timing context: the 22 ops launched one after
another (eager, CUDA events around each launch, K steps, mean), f64 at 2^28 and f32 at
2^29 elements (2 GiB planes), inputs as the reference harness draws them (magnitudes in
[1, 2), tails 2^-54 / 2^-25 below).  Prints one JSON line: op|dtype -> GB/s.
Run under TF_EW_V16=0 / all for the lean 32-byte vs 16-byte kernel A/B."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import kernels as K

K_STEPS = int(os.environ.get("SEQ_STEPS", "8"))
res = {"TF_EW_V16": os.environ.get("TF_EW_V16"), "TF_IL_LIGHT": os.environ.get("TF_IL_LIGHT"),
       "layout": os.environ.get("SEQ_LAYOUT", "split"), "gbs": {}}
for dt, n in ((torch.float64, 1 << 28), (torch.float32, 1 << 29)):
    g = torch.Generator(device="cuda").manual_seed(5)
    def plane(signed=True):
        v = torch.rand(n, dtype=dt, device="cuda", generator=g) + 1
        if signed:
            v *= (torch.rand(n, dtype=dt, device="cuda", generator=g) < 0.5).to(dt) * 2 - 1
        return v
    x0, y0, s0 = plane(), plane(), plane(False)
    sc = 2.0 ** (-54 if dt == torch.float64 else -25)
    x1, y1, s1 = x0 * sc, y0 * sc, s0 * sc
    o0, o1 = torch.empty_like(x0), torch.empty_like(x0)
    calls = []
    if os.environ.get("SEQ_LAYOUT") == "interleaved":
        from paper_1401_6235_b200 import interleaved as IL
        xp, yp, sp = (IL.from_split(K.TwofoldArray(a, b)) for a, b in ((x0, x1), (y0, y1), (s0, s1)))
        del x1, y1, s1
        op_ = torch.empty_like(xp)
        for name, spec in K.KERNELS.items():
            ins = {"22": (xp, yp), "21": (xp, y0), "11": (x0, y0), "u2": (sp, None),
                   "u1": (s0, None)}[spec.arity]
            nplanes = {"22": 6, "21": 5, "11": 4, "u2": 4, "u1": 3}[spec.arity]
            calls.append((name, IL.KERNELS[name].launch, ins + (op_,), nplanes))
        x1 = y1 = s1 = None
    else:
        for name, spec in K.KERNELS.items():
            ins = {"22": (x0, x1, y0, y1), "21": (x0, x1, y0), "11": (x0, y0),
                   "u2": (s0, s1), "u1": (s0,)}[spec.arity]
            calls.append((name, spec.loop, ins + (o0, o1), len(ins) + 2))
    for _, f, a, _np in calls:
        f(*a)
    torch.cuda.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in calls] for _ in range(K_STEPS)]
    for s in range(K_STEPS):
        for j, (_, f, a, _np) in enumerate(calls):
            ev[s][j][0].record(); f(*a); ev[s][j][1].record()
    torch.cuda.synchronize()
    tag = "f64" if dt == torch.float64 else "f32"
    for j, (name, _, a, nplanes) in enumerate(calls):
        ms = sum(ev[s][j][0].elapsed_time(ev[s][j][1]) for s in range(K_STEPS)) / K_STEPS
        res["gbs"]["%s|%s" % (name, tag)] = nplanes * n * x0.element_size() / (ms * 1e-3) / 1e9
    del x0, y0, s0, x1, y1, s1, o0, o1, calls
    torch.cuda.empty_cache()
print(json.dumps(res))
