"""The 22 elementwise kernels over the interleaved (AoS) layout.

A twofold operand or result is ONE contiguous CUDA tensor of shape (n, 2)
holding (value, error) pairs — the paper's ``twofold<T>{value, error}`` struct
 — instead of the reference's two split planes (kernels.py:3-5).
Scalar operands (the ``y`` of arity "21"/"11", the ``x`` of "11"/"u1") stay 1-D
planes.  Same names, arities, numerics (bit for bit) and validation rules as
``paper_1401_6235_b200.kernels``; outputs are always (n, 2) pair arrays.

    pairs = interleaved.from_split(x)          # TwofoldArray -> (n, 2)
    interleaved.vtadd2(pairs, pairs2, out)     # one launch, 3 streams instead of 6
    x = interleaved.to_split(out)              # (n, 2) -> TwofoldArray
"""

from __future__ import annotations


from . import _lib
from .kernels import _TABLE, RAW_OPS, TwofoldArray

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

KERNELS = {}


def _is_pairs(t):
    return (torch is not None and isinstance(t, torch.Tensor) and t.dim() == 2
            and t.shape[1] == 2)


def _desc(name, t, pairs):
    if torch is None or not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError("%s: interleaved operands must be CUDA tensors, got %r"
                         % (name, type(t).__name__))
    if pairs:
        if t.dim() != 2 or t.shape[1] != 2 or not t.is_contiguous():
            raise ValueError("%s: twofold operands must be contiguous (n, 2) pair arrays" % name)
    elif t.dim() != 1 or not t.is_contiguous():
        raise ValueError("%s: planes must be 1-D and contiguous" % name)
    if t.dtype not in (torch.float32, torch.float64):
        raise ValueError("%s: planes must be float32 or float64, got %s" % (name, t.dtype))
    return t


def _span(t):
    return t.data_ptr(), t.data_ptr() + t.numel() * t.element_size()


def _overlap(a, b):
    (a0, a1), (b0, b1) = _span(a), _span(b)
    return a.device == b.device and a0 < b1 and b0 < a1 and a1 > a0 and b1 > b0


def _make(name, arity, op):
    x_pairs = arity in ("22", "21", "u2")
    y_pairs = arity == "22"
    unary = arity in ("u2", "u1")

    def kern(*args):
        if unary:
            x, out = args
            y = None
        else:
            x, y, out = args
        ins = [_desc(name, x, x_pairs)] + ([] if unary else [_desc(name, y, y_pairs)])
        out = _desc(name, out, True)
        n = out.shape[0]
        for t in ins:
            if t.dtype != out.dtype:
                raise ValueError("%s: planes mix %s and %s" % (name, t.dtype, out.dtype))
            if t.shape[0] != n:
                raise ValueError("%s: plane lengths differ (%d vs %d)" % (name, t.shape[0], n))
            if t.device != out.device:
                raise ValueError("%s: planes live on different devices" % name)
            if _overlap(t, out):
                raise ValueError("%s: out must not alias an input" % name)
        launch(x, y, out)

    def launch(x, y, out):
        n = out.shape[0]
        if n == 0:
            return
        dev = out.device.index
        _lib.ensure_device(dev)
        dt = _lib.TF_F64 if out.dtype == torch.float64 else _lib.TF_F32
        with torch.cuda.device(dev):
            s = torch.cuda.current_stream(dev).cuda_stream
            rc = _lib.lib().tf_elementwise_il(op, dt, n, x.data_ptr(),
                                              y.data_ptr() if y is not None else None,
                                              out.data_ptr(), s)
        _lib.check(rc, name)

    kern.__name__ = kern.__qualname__ = name
    kern.__doc__ = "Interleaved-layout ``%s`` (same core as kernels.%s)." % (name, name)
    kern.launch = launch
    return kern


for _name, _arity, _op, _kind, _base, _scalar in _TABLE:
    KERNELS[_name] = _make(_name, _arity, _op)
    globals()[_name] = KERNELS[_name]
for _name, (_op, _nin) in RAW_OPS.items():
    KERNELS[_name] = _make(_name, "11" if _nin == 2 else "u1", _op)
del _name, _arity, _op, _kind, _base, _scalar


def empty_pairs(n, dtype=torch.float64 if torch else None, device="cuda"):
    """Uninitialized (n, 2) pair array."""
    return torch.empty((n, 2), dtype=dtype, device=device)


def _check_convert(name, planes, pairs):
    """Validate a split <-> interleaved conversion before any launch: the two
    1-D planes and the (n, 2) pair array share dtype, length and device, all
    contiguous CUDA tensors, and the destination overlaps no source."""
    v = _desc(name, planes[0], False)
    e = _desc(name, planes[1], False)
    p = _desc(name, pairs, True)
    n = p.shape[0]
    for t in (v, e):
        if t.dtype != p.dtype:
            raise ValueError("%s: planes mix %s and %s" % (name, t.dtype, p.dtype))
        if t.shape[0] != n:
            raise ValueError("%s: plane lengths differ (%d vs %d)" % (name, t.shape[0], n))
        if t.device != p.device:
            raise ValueError("%s: planes live on different devices" % name)
    return v, e, p, n


def from_split(x, out=None):
    """TwofoldArray of CUDA planes -> (n, 2) pair array (tf_interleave)."""
    v, e = x
    if out is None:
        _desc("from_split", v, False)
        out = torch.empty((v.shape[0], 2), dtype=v.dtype, device=v.device)
    v, e, out, n = _check_convert("from_split", (v, e), out)
    if _overlap(out, v) or _overlap(out, e):
        raise ValueError("from_split: out must not alias an input")
    if n:
        dt = _lib.TF_F64 if v.dtype == torch.float64 else _lib.TF_F32
        _lib.ensure_device(v.device.index)
        with torch.cuda.device(v.device):
            s = torch.cuda.current_stream(v.device).cuda_stream
            _lib.check(_lib.lib().tf_interleave(dt, n, v.data_ptr(), e.data_ptr(),
                                                out.data_ptr(), s), "from_split")
    return out


def to_split(pairs, out=None, kind=TwofoldArray):
    """(n, 2) pair array -> TwofoldArray of CUDA planes (tf_deinterleave)."""
    if out is None:
        _desc("to_split", pairs, True)
        n = pairs.shape[0]
        out = kind(torch.empty(n, dtype=pairs.dtype, device=pairs.device),
                   torch.empty(n, dtype=pairs.dtype, device=pairs.device))
    v, e, pairs, n = _check_convert("to_split", (out[0], out[1]), pairs)
    if _overlap(v, pairs) or _overlap(e, pairs):
        raise ValueError("to_split: out must not alias an input")
    if _overlap(v, e):
        raise ValueError("to_split: out planes overlap each other")
    if n:
        dt = _lib.TF_F64 if pairs.dtype == torch.float64 else _lib.TF_F32
        _lib.ensure_device(pairs.device.index)
        with torch.cuda.device(pairs.device):
            s = torch.cuda.current_stream(pairs.device).cuda_stream
            _lib.check(_lib.lib().tf_deinterleave(dt, n, pairs.data_ptr(), v.data_ptr(),
                                                  e.data_ptr(), s), "to_split")
    return out


__all__ = ["KERNELS", "empty_pairs", "from_split", "to_split"] + [
    row[0] for row in _TABLE]
