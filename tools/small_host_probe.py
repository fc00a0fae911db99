"""Host-pipeline probe at small/mid sizes: host_batch (vtadd2 + vtmul2 over pinned
planes) per-step time vs the raw link (one H2D of the inputs concurrent with one
D2H of the outputs, plain torch copies on two streams)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1401_6235_b200 import kernels as K

res = {"chunk_mb_env": os.environ.get("TF_HOST_CHUNK_MB"), "slots_env": os.environ.get("TF_HOST_SLOTS")}
for lg in (18, 20, 22, 24):
    n = 1 << lg
    x = [torch.rand(n, dtype=torch.float64).pin_memory().numpy() for _ in range(4)]
    outs = [K.empty_twofold(n, np.float64, device="cpu", pin_memory=True) for _ in range(2)]
    X, Y = K.TwofoldArray(x[0], x[1]), K.TwofoldArray(x[2], x[3])
    calls = [("vtadd2", X, Y, outs[0]), ("vtmul2", X, Y, outs[1])]
    for _ in range(3):
        K.host_batch(calls)
    reps = max(3, (1 << 26) // n)
    t = time.perf_counter()
    for _ in range(reps):
        K.host_batch(calls)
    dt = (time.perf_counter() - t) / reps
    # raw link: 4 planes H2D on one stream, 4 planes D2H on another, concurrently
    hin = [torch.from_numpy(a) for a in x]
    hout = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
    din = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]
    dout = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(4)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            for a, b in zip(din, hin):
                a.copy_(b, non_blocking=True)
        with torch.cuda.stream(s2):
            for a, b in zip(hout, dout):
                a.copy_(b, non_blocking=True)
        torch.cuda.synchronize()
    raw = (time.perf_counter() - t) / reps
    res[str(lg)] = {"host_batch_ms": dt * 1e3, "raw_duplex_ms": raw * 1e3,
                    "frac_of_raw": raw / dt, "gelem_ops_s": 2 * n / dt / 1e9}
print(json.dumps(res))
