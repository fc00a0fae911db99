"""Small launches of every kernel family for compute-sanitizer (memcheck /
racecheck / initcheck / synccheck): odd sizes, misaligned views, partial
tiles, multi-tile reductions with the last-CTA tree.  Exits non-zero on any
mismatch against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle as o
from paper_1401_6235_b200 import kernels as K, reduce as R, interleaved as IL, fused as F

dev = "cuda:0"
rng = np.random.default_rng(1)


def put(a, off=0):
    t = torch.empty(a.shape[0] + off, dtype=torch.float64 if a.dtype == np.float64 else torch.float32, device=dev)
    t[off:].copy_(torch.from_numpy(a))
    return t[off:]


bad = 0
for dt in (np.float64, np.float32):
    for n in (1, 37, 4099):
        for off in (0, 1):
            for name in K.KERNELS:
                spec = K.KERNELS[name]
                nin = {"22": 4, "21": 3, "11": 2, "u2": 2, "u1": 1}[spec.arity]
                ins = [rng.uniform(0.5, 2, n).astype(dt) for _ in range(nin)]
                outs = [put(np.zeros(n, dt), off) for _ in range(2)]
                spec.loop(*[put(a, off) for a in ins], *outs)
                w = o.elementwise(name, *ins)
                if not (np.array_equal(outs[0].cpu().numpy(), w[0]) and np.array_equal(outs[1].cpu().numpy(), w[1])):
                    bad += 1
                    print("mismatch", name, dt, n, off)
    for n in (1, 5, 65536 * 3 + 7):
        x = rng.uniform(-1, 1, n).astype(dt)
        y = rng.uniform(-1, 1, n).astype(dt)
        for rop in ("sum", "dot", "sum2"):
            if rop == "sum":
                z = R.vtsum(put(x))
            elif rop == "dot":
                z = R.vtdot(put(x), put(y))
            else:
                z = R.vtsum2((put(x), put(y)))
            g = R.geometry(dt)
            w = o.reduce(rop, x, None if rop == "sum" else y, geometry=g)
            if (z.value, z.error) != (float(w[0]), float(w[1])):
                bad += 1
                print("reduce mismatch", rop, dt, n)
    xs = rng.uniform(0.9, 1.1, 999).astype(dt)
    out = K.empty_twofold(999, torch.float64 if dt == np.float64 else torch.float32)
    for cf in (R.binomial_coeffs(20), [0.5, -0.0, 3.0, -0.0, 1.0, -2.0, 0.0]):
        R.vthorner(cf, put(xs), out)
        w = o.horner(cf, xs)
        if not (np.array_equal(out.value.cpu().numpy(), w[0]) and
                np.array_equal(out.error.cpu().numpy(), w[1])):
            bad += 1
            print("horner mismatch", dt, len(cf))
    p = IL.from_split(K.TwofoldArray(put(xs), put(xs)))
    po = torch.empty_like(p)
    IL.vtadd2(p, p, po)
    F.vtaxpy(K.TwofoldArray(put(xs), put(xs)), K.TwofoldArray(put(xs), put(xs)), K.TwofoldArray(put(xs), put(xs)))
# multi-tile elementwise launches (chunked CTAs; on the TMA-staged path several
# shared-memory refills per CTA), misaligned head and a tail, every op
for dt in (np.float64, np.float32):
    n = (1 << 23) + 4099
    for name in K.KERNELS:
        spec = K.KERNELS[name]
        nin = {"22": 4, "21": 3, "11": 2, "u2": 2, "u1": 1}[spec.arity]
        ins = [rng.uniform(0.5, 2, n).astype(dt) for _ in range(nin)]
        outs = [put(np.zeros(n, dt), 1) for _ in range(2)]
        spec.loop(*[put(a, 1) for a in ins], *outs)
        w = o.elementwise(name, *ins)
        if not (np.array_equal(outs[0].cpu().numpy(), w[0]) and np.array_equal(outs[1].cpu().numpy(), w[1])):
            bad += 1
            print("mismatch (multi-tile)", name, dt, n)
        del ins, outs, w
# device batch (one launch, shared planes) and reduction pairs (one pass)
for dt in (np.float64, np.float32):
    for n in (37, 4099, 3 * 65536 + 11):
        for off in (0, 1):
            ins = [rng.uniform(0.5, 2, n).astype(dt) for _ in range(4)]
            P = [put(a, off) for a in ins]
            X, Y = K.TwofoldArray(P[0], P[1]), K.TwofoldArray(P[2], P[3])
            outs = [K.TwofoldArray(put(np.zeros(n, dt), off), put(np.zeros(n, dt), off)) for _ in range(3)]
            K.batch([("vtadd2", X, Y, outs[0]), ("vtdiv2", X, Y, outs[1]), ("vtsqrt1", X, outs[2])])
            for name, o_, w in (("vtadd2", outs[0], o.elementwise("vtadd2", *ins)),
                                ("vtdiv2", outs[1], o.elementwise("vtdiv2", *ins)),
                                ("vtsqrt1", outs[2], o.elementwise("vtsqrt1", ins[0], ins[1]))):
                if not (np.array_equal(o_.value.cpu().numpy(), w[0]) and
                        np.array_equal(o_.error.cpu().numpy(), w[1])):
                    bad += 1
                    print("batch mismatch", name, dt, n, off)
            zd, zs = R.batch([("vtdot", P[0], P[2]), ("vtsum", P[0])])
            geo = R.geometry(dt)
            wd = o.reduce("dot", ins[0], ins[2], geometry=geo)
            wsum = o.reduce("sum", ins[0], geometry=geo)
            if tuple(zd) != (float(wd[0]), float(wd[1])) or tuple(zs) != (float(wsum[0]), float(wsum[1])):
                bad += 1
                print("reduce pair mismatch", dt, n, off)
# host-plane pipeline (pinned and pageable), several chunks
for dt in (np.float64, np.float32):
    n = 3 * (1 << 18) + 5
    ins = [rng.uniform(0.5, 2, n).astype(dt) for _ in range(4)]
    out = K.empty_twofold(n, dt, device="cpu")
    K.vtdiv2(K.TwofoldArray(ins[0], ins[1]), K.TwofoldArray(ins[2], ins[3]), out)
    w = o.elementwise("vtdiv2", *ins)
    if not (np.array_equal(out.value, w[0]) and np.array_equal(out.error, w[1])):
        bad += 1
        print("host path mismatch", dt)
# pinned host planes (small: the zero-copy kernel by default; TF_HOST_ZEROCOPY_MB
# selects the staged pipeline or forces zero-copy), unaligned interior views
for dt in (np.float64, np.float32):
    n = 3 * (1 << 16) + 7
    tdt = torch.float64 if dt == np.float64 else torch.float32
    pins = [torch.from_numpy(rng.uniform(0.5, 2, n + 3).astype(dt)).pin_memory().numpy()[k % 3:k % 3 + n]
            for k in range(4)]
    outs = [torch.empty(n + 1, dtype=tdt).pin_memory().numpy()[1:] for _ in range(4)]
    X, Y = K.TwofoldArray(pins[0], pins[1]), K.TwofoldArray(pins[2], pins[3])
    K.host_batch([("vtdiv2", X, Y, K.TwofoldArray(outs[0], outs[1])),
                  ("vtadd2", X, Y, K.TwofoldArray(outs[2], outs[3]))])
    for name, a, b in (("vtdiv2", outs[0], outs[1]), ("vtadd2", outs[2], outs[3])):
        w = o.elementwise(name, *pins)
        if not (np.array_equal(a, w[0]) and np.array_equal(b, w[1])):
            bad += 1
            print("pinned host path mismatch", name, dt)
torch.cuda.synchronize()
print("sanitize smoke done, mismatches:", bad)
sys.exit(1 if bad else 0)
