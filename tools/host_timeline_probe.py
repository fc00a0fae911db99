"""GPU timeline of one host_batch call (CUPTI via torch.profiler): when each
H2D/D2H copy and kernel of the pipeline runs, per stream."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
from paper_1401_6235_b200 import kernels as K

n = 1 << int(os.environ.get("LGN", "20"))
x = [torch.rand(n, dtype=torch.float64).pin_memory().numpy() for _ in range(4)]
outs = [K.empty_twofold(n, np.float64, device="cpu", pin_memory=True) for _ in range(2)]
X, Y = K.TwofoldArray(x[0], x[1]), K.TwofoldArray(x[2], x[3])
calls = [("vtadd2", X, Y, outs[0]), ("vtmul2", X, Y, outs[1])]
for _ in range(5):
    K.host_batch(calls)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    K.host_batch(calls)
    torch.cuda.synchronize()
path = "gpurun_out/timeline_%d.json" % n
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
rows = []
for e in ev:
    if e.get("ph") != "X":
        continue
    cat = e.get("cat", "")
    if cat in ("gpu_memcpy", "kernel", "cuda_runtime", "cuda_driver"):
        rows.append((e["ts"], e.get("dur", 0), cat, e["name"][:40], e.get("args", {}).get("stream", e.get("tid"))))
rows.sort()
t0 = rows[0][0] if rows else 0
for r in rows:
    print("%9.1f %8.1f %-13s %-40s %s" % (r[0] - t0, r[1], r[2], r[3], r[4]))
