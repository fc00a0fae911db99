"""Zero-copy probe: the device batch kernel reading and writing pinned HOST
planes directly over PCIe (UVA-mapped), vs the staged host_batch pipeline."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1401_6235_b200 import _lib
from paper_1401_6235_b200 import kernels as K

res = {}
for lg in (18, 20, 21, 22, 23, 24, 27):
    n = 1 << lg
    pl = [torch.rand(n, dtype=torch.float64).pin_memory() for _ in range(8)]
    outs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(10)]
    npl = [p.numpy() for p in pl]
    T = K.TwofoldArray
    X, Y, D, Q = T(npl[0], npl[1]), T(npl[2], npl[3]), T(npl[4], npl[5]), T(npl[6], npl[7])
    O = [T(outs[2 * i].numpy(), outs[2 * i + 1].numpy()) for i in range(5)]
    calls = [("vtadd2", X, Y, O[0]), ("vtsub2", X, Y, O[1]), ("vtmul2", X, Y, O[2]),
             ("vtdiv2", X, D, O[3]), ("vtsqrt1", Q, O[4])]
    reps = max(2, (1 << 27) // n)
    K.host_batch(calls)
    t = time.perf_counter()
    for _ in range(reps):
        K.host_batch(calls)
    staged = (time.perf_counter() - t) / reps
    ref = [o.clone() for o in outs]
    ops, ins, outp, first, _ = K._parse_batch(calls, "zc")
    L = _lib.lib()
    arr = (ctypes.c_int * 5)(*ops)
    s = torch.cuda.current_stream().cuda_stream
    pin, pout = _lib.ptr_array(ins), _lib.ptr_array(outp)
    for o in outs:
        o.zero_()
    _lib.check(L.tf_elementwise_batch(5, arr, 1, n, pin, pout, s), "zc")
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(ref, outs))
    t = time.perf_counter()
    for _ in range(reps):
        L.tf_elementwise_batch(5, arr, 1, n, pin, pout, s)
    torch.cuda.synchronize()
    zc = (time.perf_counter() - t) / reps
    res[str(lg)] = {"staged_ms": staged * 1e3, "zerocopy_ms": zc * 1e3, "same_bits": same,
                    "staged_gelem_ops": 5 * n / staged / 1e9, "zc_gelem_ops": 5 * n / zc / 1e9,
                    "zc_link_gbs": 18 * 8 * n / zc / 1e9}
    del pl, outs
print(json.dumps(res, indent=1))
