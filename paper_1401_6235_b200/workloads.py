"""Seeded synthetic workloads with BASELINE.json's distributions (device-generated).

Used by bench.py and the full-size GPU parity tests.  Element i of a plane
depends only on (seed, offset + i) (counter-based splitmix64 in tf_fill), so a
rank's shard of a global array is generated independently of the rank count.

Distributions (BASELINE.json configs):
  config1  f64 add/mul: heads U[-1,1], tails head*2^-53*U[-1,1]
  config2  f64 add/sub/mul/div/sqrt: heads ±2^U[-20,20]; divisors 2^U[-10,10];
           sqrt inputs 2^U[-20,20]; tails head*2^-53*U[-1,1]
  config3  f32 add/mul/div: heads U[-1,1]; tails head*2^-24*U[-1,1]; divisors U[0.5,2]
  config5  Horner points U[0.9,1.1]
(config 4 uses the host ORO-style generator tf_gen_dot_host.)
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


__all__ = ["fill", "dists", "PlaneSet", "UNIFORM", "LOGU_SIGNED", "LOGU_POS", "TAIL"]
