"""A/B timing of split-layout elementwise kernels on BASELINE config-2/3 planes.

    TF_LIB_PATH=<variant .so> python tools/ew_ab.py [--ops vtsqrt1,vtadd2] [--n 268435456]

Each op: K eager launches on the bench's own planes (workloads.PlaneSet, the
BASELINE distributions), CUDA events around every launch; prints one JSON line
with mean / median GB/s per op and the library path, so several variants can be
run back to back in separate processes and compared.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1401_6235_b200 import _lib, kernels as K, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ops", default="vtadd2,vtsqrt1")
ap.add_argument("--n", type=int, default=1 << 28)
ap.add_argument("--config", default="config2")
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
dt = torch.float64 if a.config != "config3" else torch.float32
esz = 8 if dt == torch.float64 else 4
ps = W.PlaneSet(a.config, a.n, dt, 0)
out = K.empty_twofold(a.n, dt)
res = {"lib": str(_lib.LIB_PATH), "n": a.n}
for name in a.ops.split(","):
    planes = ps.planes(name)
    loop = K.KERNELS[name].loop
    # warm up for ~2 s so the SM clock has left its idle state (a compute-heavy
    # op timed right after start-up runs at a ramping clock)
    import time
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 2.0:
        for _ in range(10):
            loop(*planes, out.value, out.error)
        torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.reps)]
    torch.cuda.synchronize()
    for e0, e1 in ev:
        e0.record()
        loop(*planes, out.value, out.error)
        e1.record()
    torch.cuda.synchronize()
    ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        res.setdefault("sm_mhz_after", {})[name] = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:
        pass
    nbytes = (len(planes) + 2) * esz * a.n
    res[name] = {"mean_gbs": nbytes / (statistics.mean(ms) * 1e-3) / 1e9,
                 "median_gbs": nbytes / (statistics.median(ms) * 1e-3) / 1e9,
                 "best_gbs": nbytes / (min(ms) * 1e-3) / 1e9}
print(json.dumps(res), flush=True)
