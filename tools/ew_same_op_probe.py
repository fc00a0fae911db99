"""One op repeated back to back (as gpubench replays it) in three timings: events around every
launch (mean and best) and a CUDA graph of 16 launches replayed 7 times (mean and best replay).
f64, 2^27 elements, reference-harness inputs.  Run under TF_EW_V16=0 / all."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import kernels as K

n = 1 << 27
g = torch.Generator(device="cuda").manual_seed(5)
pl = [torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 1 for _ in range(4)]
pl[1] *= 2.0 ** -54
pl[3] *= 2.0 ** -54
o0, o1 = torch.empty_like(pl[0]), torch.empty_like(pl[0])
res = {"TF_EW_V16": os.environ.get("TF_EW_V16"), "gbs": {}}
for name, args in (("vtadd2", pl + [o0, o1]), ("vtdiv2", pl + [o0, o1]), ("vtsqrt1", pl[:2] + [o0, o1])):
    f = K.KERNELS[name].loop
    nbytes = len(args) * n * 8
    for _ in range(5):
        f(*args)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
    for a, b in ev:
        a.record(); f(*args); b.record()
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for a, b in ev]
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for _ in range(16):
            f(*args)
    gr.replay(); torch.cuda.synchronize()
    rs = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        with torch.cuda.stream(st):
            gr.replay()
        b.record(st); b.synchronize()
        rs.append(a.elapsed_time(b) / 16)
    gb = lambda ms: round(nbytes / (ms * 1e-3) / 1e9)
    res["gbs"][name] = {"eager_mean": gb(sum(ts) / len(ts)), "eager_best": gb(min(ts)),
                        "graph_mean": gb(sum(rs) / len(rs)), "graph_best": gb(min(rs))}
print(json.dumps(res))
