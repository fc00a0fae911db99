"""vtadd2 / vtsqrt1 over views that share their alignment modulo 16 bytes but not modulo 32
(plane k offset by 2k f64 elements): the 16-byte kernel vectorises them; with TF_EW_V16=0
they take the scalar path.  Prints GB/s (CUDA events, mean of 10 after warm-up)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import kernels as K

n = 1 << 27
res = {"TF_EW_V16": os.environ.get("TF_EW_V16"), "gbs": {}}
for label, offs in (("aligned", [0] * 6), ("half-aligned", [0, 2, 4, 6, 0, 2]), ("mixed", [0, 1, 2, 0, 1, 2])):
    pl = [torch.rand(n + 8, dtype=torch.float64, device="cuda")[o:o + n] + 1 for o in offs]
    for name, args in (("vtadd2", pl), ("vtsqrt1", pl[:2] + pl[4:])):
        f = K.KERNELS[name].loop
        for _ in range(3):
            f(*args)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            f(*args)
        b.record(); b.synchronize()
        res["gbs"]["%s %s" % (name, label)] = len(args) * n * 8 * 10 / (a.elapsed_time(b) * 1e-3) / 1e9
print(json.dumps(res))
