"""Debug: TMA-staged elementwise path vs torch IEEE ops (z0 plane) at several sizes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_6235_b200 import kernels as K, workloads as W

for n in [1 << 20, 1 << 24, 1 << 26, 1 << 27, 1 << 28]:
    ps = W.PlaneSet("config2", n, torch.float64, 0)
    out = K.empty_twofold(n, torch.float64)
    for name in ["vtsqrt1", "vtadd2"]:
        pl = ps.planes(name)
        out.value.fill_(float("nan"))
        K.KERNELS[name].loop(*pl, out.value, out.error)
        torch.cuda.synchronize()
        want = torch.sqrt(pl[0]) if name == "vtsqrt1" else pl[0] + pl[2]
        bad = (out.value.view(torch.int64) != want.view(torch.int64)).nonzero().flatten()
        msg = "%s n=2^%d bad=%d" % (name, n.bit_length() - 1, bad.numel())
        if bad.numel():
            b = bad.cpu()
            vec = b // 4
            tile = vec // 256
            msg += " first=%s tiles=%s ntiles_bad=%d thr=%s nan=%d" % (
                b[:4].tolist(), tile.unique()[:8].tolist(), tile.unique().numel(),
                (vec % 256).unique()[:8].tolist(), int(torch.isnan(out.value[bad]).sum()))
        print(msg, flush=True)
    del ps, out
    torch.cuda.empty_cache()
