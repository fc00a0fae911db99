"""split <-> interleaved conversion kernels at bench sizes (CUDA events, best/mean of
reps after warm-up; inputs far larger than L2).  Bytes per element: 2 planes in +
1 pair array out = 4*sizeof(T).  Usage: python tools/convert_bench.py [--lg 27 28]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import interleaved as IL

ap = argparse.ArgumentParser()
ap.add_argument("--lg", type=int, nargs="*", default=[27, 28])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
res = {"TF_CONV_LEAN": os.environ.get("TF_CONV_LEAN"), "rows": []}
for dt in (torch.float64, torch.float32):
    for lg in a.lg:
        n = (1 << lg) * (2 if dt == torch.float32 else 1)
        v = torch.rand(n, dtype=dt, device="cuda")
        e = torch.rand(n, dtype=dt, device="cuda")
        pairs = torch.empty((n, 2), dtype=dt, device="cuda")
        v2, e2 = torch.empty_like(v), torch.empty_like(e)
        from paper_1401_6235_b200.kernels import TwofoldArray
        x = TwofoldArray(v, e)
        o = TwofoldArray(v2, e2)
        for name, fn in (("interleave", lambda: IL.from_split(x, pairs)),
                         ("deinterleave", lambda: IL.to_split(pairs, o))):
            for _ in range(3):
                fn()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(a.reps)]
            for s, t in ev:
                s.record(); fn(); t.record()
            torch.cuda.synchronize()
            ts = [s.elapsed_time(t) for s, t in ev]
            nbytes = 4 * n * v.element_size()
            res["rows"].append({"kernel": name, "dtype": str(dt).split(".")[-1], "n": n,
                                "ms_mean": sum(ts) / len(ts), "ms_best": min(ts),
                                "gbs_mean": nbytes / (sum(ts) / len(ts) * 1e-3) / 1e9,
                                "gbs_best": nbytes / (min(ts) * 1e-3) / 1e9})
        assert torch.equal(v2, v) and torch.equal(e2, e)
        del v, e, pairs, v2, e2
        torch.cuda.empty_cache()
print(json.dumps(res))
