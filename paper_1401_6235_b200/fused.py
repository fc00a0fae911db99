"""Fused twofold expression kernels over n independent instances.

The reference's application studies chain scalar twofold operations
(/root/reference/pkg/src/twofold/demos.py): Gauss elimination of a 3x3 system
(demos.py:153-199, the update ``a[i][j] = tsub(a[i][j], tmul(m, a[k][j]))`` at
:182-184) and the school formula for quadratic roots (demos.py:211-238).  These
kernels run the same chains, op for op, over batches of independent instances,
with every intermediate kept in registers — bit-identical to composing the
elementwise kernels, at a fraction of their HBM traffic.

    vtaxpy(a, x, y, out)            out = tadd(tmul(a, x), y)
    vtsubmul(c, a, b, out)          out = tsub(c, tmul(a, b))
    vtquadratic(a, b, c) -> (d, x0, x1)      TwofoldArrays of the demo's d, x0, x1
    vtgauss3(A, f) -> x             A: TwofoldArray of (3, 3, n) planes, f: (3, n)

All operands are TwofoldArrays of CUDA tensors of one dtype.
"""

from __future__ import annotations

from . import _lib
from .kernels import TwofoldArray

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

FAXPY, FSUBMUL, FQUAD, FGAUSS3 = 0, 1, 2, 3


def _planes(name, tfs, shape=None):
    out = []
    for t in tfs:
        for p in t:
            if torch is None or not isinstance(p, torch.Tensor) or not p.is_cuda:
                raise ValueError("%s: planes must be CUDA tensors, got %r" % (name, type(p).__name__))
            if not p.is_contiguous():
                raise ValueError("%s: planes must be contiguous" % name)
            if p.dtype not in (torch.float32, torch.float64):
                raise ValueError("%s: planes must be float32 or float64, got %s" % (name, p.dtype))
            out.append(p)
    first = out[0]
    for p in out[1:]:
        if p.dtype != first.dtype:
            raise ValueError("%s: planes mix %s and %s" % (name, first.dtype, p.dtype))
        if p.device != first.device:
            raise ValueError("%s: planes live on different devices" % name)
    return out


def _launch(name, fop, n, ins, outs):
    if n == 0:
        return
    dev = ins[0].device.index
    _lib.ensure_device(dev)
    dt = _lib.TF_F64 if ins[0].dtype == torch.float64 else _lib.TF_F32
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev).cuda_stream
        rc = _lib.lib().tf_fused(fop, dt, n, _lib.ptr_array([p.data_ptr() for p in ins]),
                                 _lib.ptr_array([p.data_ptr() for p in outs]), s)
    _lib.check(rc, name)


def _same_len(name, planes, n):
    for p in planes:
        if p.dim() != 1 or p.shape[0] != n:
            raise ValueError("%s: plane lengths differ" % name)


def _no_alias(name, ins, outs):
    def span(t):
        return t.data_ptr(), t.data_ptr() + t.numel() * t.element_size()

    for o in outs:
        a0, a1 = span(o)
        for i in ins:
            b0, b1 = span(i)
            if a0 < b1 and b0 < a1:
                raise ValueError("%s: out must not alias an input" % name)


def _empty_like(p, kind=TwofoldArray):
    return kind(torch.empty_like(p), torch.empty_like(p))


def vtaxpy(a, x, y, out=None):
    """out = tadd(tmul(a, x), y), elementwise (arith.py:86-94 then 61-64)."""
    ins = _planes("vtaxpy", (a, x, y))
    out = out if out is not None else _empty_like(ins[0])
    outs = _planes("vtaxpy", (out,))
    n = ins[0].shape[0]
    _same_len("vtaxpy", ins + outs, n)
    _no_alias("vtaxpy", ins, outs)
    _launch("vtaxpy", FAXPY, n, ins, outs)
    return out


def vtsubmul(c, a, b, out=None):
    """out = tsub(c, tmul(a, b)): the elimination update of demos.py:182-184."""
    ins = _planes("vtsubmul", (c, a, b))
    out = out if out is not None else _empty_like(ins[0])
    outs = _planes("vtsubmul", (out,))
    n = ins[0].shape[0]
    _same_len("vtsubmul", ins + outs, n)
    _no_alias("vtsubmul", ins, outs)
    _launch("vtsubmul", FSUBMUL, n, ins, outs)
    return out


def vtquadratic(a, b, c, out=None):
    """Roots of a·x² + b·x + c by the school formula (demos.py:222-229).

    Returns (d, x0, x1) as TwofoldArrays: d = tsqrt(b² − 4ac),
    x0 = (−b − d)/(2a), x1 = (−b + d)/(2a), every step twofold."""
    ins = _planes("vtquadratic", (a, b, c))
    n = ins[0].shape[0]
    if out is None:
        out = tuple(_empty_like(ins[0]) for _ in range(3))
    outs = _planes("vtquadratic", out)
    _same_len("vtquadratic", ins + outs, n)
    _no_alias("vtquadratic", ins, outs)
    _launch("vtquadratic", FQUAD, n, ins, outs)
    return out


def vtgauss3(A, f, out=None):
    """Solve n independent 3x3 twofold systems by the reference's naive Gauss
    elimination (demos.py:175-192).  A = TwofoldArray of (3, 3, n) planes (row
    major, contiguous), f = TwofoldArray of (3, n); returns x as (3, n) planes."""
    av, ae = A
    fv, fe = f
    for t, shape in ((av, 3), (ae, 3), (fv, 2), (fe, 2)):
        if torch is None or not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError("vtgauss3: planes must be CUDA tensors")
        if t.dim() != shape or not t.is_contiguous():
            raise ValueError("vtgauss3: A planes must be contiguous (3, 3, n), f planes (3, n)")
    n = av.shape[-1]
    if av.shape != (3, 3, n) or ae.shape != av.shape or fv.shape != (3, n) or fe.shape != (3, n):
        raise ValueError("vtgauss3: A planes must be (3, 3, n), f planes (3, n)")
    if out is None:
        out = TwofoldArray(torch.empty_like(fv), torch.empty_like(fe))
    ins = _planes("vtgauss3", (A, f))
    outs = _planes("vtgauss3", (out,))
    _no_alias("vtgauss3", ins, outs)
    _launch("vtgauss3", FGAUSS3, n, ins, outs)
    return out


__all__ = ["vtaxpy", "vtsubmul", "vtquadratic", "vtgauss3"]
