"""Seeded synthetic workloads with BASELINE.json's distributions (device-generated).

Used by bench.py and the full-size GPU parity tests.  Element i of a plane
depends only on (seed, offset + i) (counter-based splitmix64 in tf_fill), so a
rank's shard of a global array is generated independently of the rank count.

Distributions (BASELINE.json configs):
  config1  f64 add/mul: heads U[-1,1], tails head*2^-53*U[-1,1]
  config2  f64 add/sub/mul/div/sqrt: heads ±2^U[-20,20]; divisors 2^U[-10,10];
           sqrt inputs 2^U[-20,20]; tails head*2^-53*U[-1,1]
  config3  f32 add/mul/div: heads U[-1,1]; tails head*2^-24*U[-1,1]; divisors U[0.5,2]
  config4  f64 dot x.y and sum of p, cond 1e16: blocked Ogita-Rump-Oishi-style
           generators (tf_gen_ill, csrc/gen_ill.cu): per 65536-element block
           half the terms have random exponents in [-50, 50], the rest cancel
           the block's running value; every block ends on a calibrated
           positive target, so any run of whole blocks has cond 1e16
  config5  Horner points U[0.9,1.1]
"""

from __future__ import annotations

from . import _lib

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

# fill kinds of tf_fill
UNIFORM, LOGU_SIGNED, LOGU_POS, TAIL = 0, 1, 2, 3


def fill(t, kind, seed, offset, lo, hi, head=None):
    """Fill CUDA tensor t in place (asynchronous on the current stream)."""
    dt = _lib.TF_F64 if t.dtype == torch.float64 else _lib.TF_F32
    _lib.ensure_device(t.device.index)
    with torch.cuda.device(t.device):
        rc = _lib.lib().tf_fill(dt, kind, t.numel(), seed, offset, lo, hi,
                                head.data_ptr() if head is not None else None, t.data_ptr(),
                                torch.cuda.current_stream(t.device).cuda_stream)
    _lib.check(rc, "tf_fill")
    return t


# BASELINE configs[3]: the ill-conditioned dot and sum inputs
C4_N = 1 << 30
C4_COND = 1e16
C4_SEED = 4242
C4_EMIN, C4_EMAX = -50, 50
GEN_BLOCK = 65536  # TF_GEN_BLOCK
GEN_DOT, GEN_SUM = 0, 1


def gen_ill(kind, x, y=None, n_total=None, first=0, cond=C4_COND, seed=C4_SEED,
            emin=C4_EMIN, emax=C4_EMAX):
    """Global elements [first, first + len(x)) of the config-4 problem of
    ``n_total`` elements (default len(x)) into CUDA tensor x (and y for the
    dot), asynchronous on the current stream (tf_gen_ill).  numpy planes are
    filled on the host threads instead (tf_gen_ill_host), with the same bits."""
    import numpy as np

    count = x.shape[0]
    n_total = count if n_total is None else n_total
    if isinstance(x, np.ndarray):
        rc = _lib.lib().tf_gen_ill_host(kind, n_total, first, count, cond, seed, emin, emax,
                                        x.ctypes.data, y.ctypes.data if y is not None else None, 0)
        _lib.check(rc, "tf_gen_ill_host")
        return x, y
    _lib.ensure_device(x.device.index)
    with torch.cuda.device(x.device):
        rc = _lib.lib().tf_gen_ill(kind, n_total, first, count, cond, seed, emin, emax,
                                   x.data_ptr(), y.data_ptr() if y is not None else None,
                                   torch.cuda.current_stream(x.device).cuda_stream)
    _lib.check(rc, "tf_gen_ill")
    return x, y


def config4_planes(n_total, first, count, device):
    """(x, y, p) CUDA planes of rank slice [first, first + count) of the config-4
    problem: x.y is the ill-conditioned dot, p the ill-conditioned sum."""
    x = torch.empty(count, dtype=torch.float64, device=device)
    y = torch.empty(count, dtype=torch.float64, device=device)
    p = torch.empty(count, dtype=torch.float64, device=device)
    gen_ill(GEN_DOT, x, y, n_total=n_total, first=first)
    gen_ill(GEN_SUM, p, n_total=n_total, first=first)
    return x, y, p


def dists(config):
    """op -> list of (kind, lo, hi) per input plane; TAIL derives from the previous plane."""
    if config == "config1":
        head, tail = (UNIFORM, -1.0, 1.0), (TAIL, -53.0, 0.0)
        return {"vtadd2": [head, tail, head, tail], "vtmul2": [head, tail, head, tail]}
    if config == "config2":
        head, tail = (LOGU_SIGNED, -20.0, 20.0), (TAIL, -53.0, 0.0)
        div, pos = (LOGU_POS, -10.0, 10.0), (LOGU_POS, -20.0, 20.0)
        return {"vtadd2": [head, tail, head, tail], "vtsub2": [head, tail, head, tail],
                "vtmul2": [head, tail, head, tail], "vtdiv2": [head, tail, div, tail],
                "vtsqrt1": [pos, tail]}
    if config == "config3":
        head, tail, div = (UNIFORM, -1.0, 1.0), (TAIL, -24.0, 0.0), (UNIFORM, 0.5, 2.0)
        return {"vtadd2": [head, tail, head, tail], "vtmul2": [head, tail, head, tail],
                "vtdiv2": [head, tail, div, tail]}
    raise ValueError("unknown config %r" % config)


class PlaneSet:
    """Device planes for a config's ops, shared where the distributions agree
    (x and y never share: the plane position is part of the key)."""

    def __init__(self, config, n, dtype, device, offset=0, seed0=1000):
        self.config, self.n, self.dtype, self.device = config, n, dtype, device
        self.offset, self.seed0 = offset, seed0
        self.cache = {}
        self.keys = {}
        self.d = dists(config)

    def planes(self, op):
        out, keys = [], []
        for k, (kind, lo, hi) in enumerate(self.d[op]):
            key = (k, kind, lo, hi, keys[k - 1] if kind == TAIL else None)
            keys.append(key)
            if key not in self.cache:
                t = torch.empty(self.n, dtype=self.dtype, device=self.device)
                fill(t, kind, self.seed0 + 17 * len(self.cache), self.offset, lo, hi,
                     out[k - 1] if kind == TAIL else None)
                self.cache[key] = t
            out.append(self.cache[key])
        self.keys[op] = keys
        return out


__all__ = ["fill", "dists", "PlaneSet", "UNIFORM", "LOGU_SIGNED", "LOGU_POS", "TAIL",
           "gen_ill", "config4_planes", "GEN_DOT", "GEN_SUM", "C4_N", "C4_COND", "C4_SEED"]
