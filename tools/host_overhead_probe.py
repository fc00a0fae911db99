"""Where the fixed cost of a small host_batch call goes: Python validation vs the
library call, at n = 1 (pure overhead) and 2^18."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1401_6235_b200 import _lib
from paper_1401_6235_b200 import kernels as K


def best(f, reps=200):
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t)
    ts.sort()
    return {"min_us": ts[0] * 1e6, "med_us": ts[len(ts) // 2] * 1e6}


res = {}
for n in (1, 1 << 18):
    x = [torch.rand(n, dtype=torch.float64).pin_memory().numpy() for _ in range(4)]
    outs = [K.empty_twofold(n, np.float64, device="cpu", pin_memory=True) for _ in range(2)]
    X, Y = K.TwofoldArray(x[0], x[1]), K.TwofoldArray(x[2], x[3])
    calls = [("vtadd2", X, Y, outs[0]), ("vtmul2", X, Y, outs[1])]
    K.host_batch(calls)
    ops, ins, outp, first, _ = K._parse_batch(calls, "p")
    L = _lib.lib()
    arr_ops = (ctypes.c_int * 2)(*ops)
    pin, pout = _lib.ptr_array(ins), _lib.ptr_array(outp)
    r = {"parse": best(lambda: K._parse_batch(calls, "p")),
         "ctypes_call": best(lambda: L.tf_elementwise_host_batch(2, arr_ops, 1, n, pin, pout, 0)),
         "host_batch": best(lambda: K.host_batch(calls)),
         "vtadd2_host": best(lambda: K.vtadd2(X, Y, outs[0]))}
    res[str(n)] = r
print(json.dumps(res))
