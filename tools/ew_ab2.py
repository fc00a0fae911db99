"""Interleaved in-process A/B of library variants on one op (same power/clock state).

    python tools/ew_ab2.py --op vtsqrt1 --libs a.so,b.so,... [--n 2^28] [--rounds 8]

Loads every variant .so side by side (ctypes, RTLD_LOCAL: each has its own static
CUDA runtime), then alternates: each round times K launches of the op per
variant with CUDA events on one stream.  Prints one JSON line: per variant the
median GB/s over rounds and the register count is left to cuobjdump.
"""
import argparse, ctypes, json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import _lib, kernels as K, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="vtsqrt1")
ap.add_argument("--libs", required=True)
ap.add_argument("--n", type=int, default=1 << 28)
ap.add_argument("--config", default="config2")
ap.add_argument("--rounds", type=int, default=8)
ap.add_argument("--k", type=int, default=10)
a = ap.parse_args()
dt = torch.float64 if a.config != "config3" else torch.float32
esz = 8 if dt == torch.float64 else 4
ps = W.PlaneSet(a.config, a.n, dt, 0)
planes = ps.planes(a.op)
out = K.empty_twofold(a.n, dt)
op = K.KERNELS[a.op].core
libs = []
for path in a.libs.split(","):
    L = ctypes.CDLL(path)
    L.tf_elementwise.restype = ctypes.c_int
    L.tf_elementwise.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                 ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.c_void_p]
    L.tf_last_error.restype = ctypes.c_char_p
    assert L.tf_selftest(0) == 0, L.tf_last_error()
    libs.append((path, L))
ins = _lib.ptr_array([p.data_ptr() for p in planes])
outs = _lib.ptr_array([out.value.data_ptr(), out.error.data_ptr()])
stream = None  # the legacy default stream: valid in every runtime copy (torch records its events there too)
dtid = _lib.TF_F64 if dt == torch.float64 else _lib.TF_F32
t0 = time.perf_counter()
while time.perf_counter() - t0 < 2.0:  # clocks out of idle, power state settled
    for _, L in libs:
        rc = L.tf_elementwise(op, dtid, a.n, ins, outs, stream)
        assert rc == 0, (rc, L.tf_last_error())
    torch.cuda.synchronize()
res = {p: [] for p, _ in libs}
nbytes = (len(planes) + 2) * esz * a.n
for r in range(a.rounds):
    order = libs if r % 2 == 0 else libs[::-1]
    for path, L in order:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.k):
            L.tf_elementwise(op, dtid, a.n, ins, outs, stream)
        e1.record()
        torch.cuda.synchronize()
        res[path].append(nbytes * a.k / (e0.elapsed_time(e1) * 1e-3) / 1e9)
print(json.dumps({"op": a.op, "n": a.n, "gbs_median": {p.split("/")[-2]: statistics.median(v) for p, v in res.items()},
                  "gbs_all": {p.split("/")[-2]: [round(x) for x in v] for p, v in res.items()}}), flush=True)
