"""Twofold reductions (sum, twofold-input sum, dot) and twofold Horner on B200.

The reference has no array API for these (its only reduction is the serial
``_accumulate`` fold of ``_tadd``, demos.py:107-113).  They are composed from
the reference cores — ``_tadd1`` (arith.py:67-71), ``_tadd`` (arith.py:61-64),
``_two_prod`` (fp_core.py:170-173), ``_tmul1`` (arith.py:97-101) — in the
canonical order documented in DESIGN.md, which the CPU oracle restates, so
results are bit-exact against it and bit-identical for any number of shards.

    vtsum(x)          -> Twofold   Σ x_i           (z0 = plain sum in that order)
    vtsum2(x)         -> Twofold   Σ (x0_i + x1_i) for a TwofoldArray x
    vtdot(x, y)       -> Twofold   Σ x_i * y_i
    vthorner(c, x, out)            twofold Horner of Σ c_k x^k at every x_i

Reductions return a ``Twofold`` of Python floats (one device->host read of 16
bytes) unless ``out=`` (a 2-element CUDA tensor) is given, in which case they
stay asynchronous on the current stream.
"""

from __future__ import annotations

import ctypes
from collections import namedtuple

import numpy as np

from . import _lib
from .kernels import TwofoldArray, _check, _describe, _dtype_id

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

Twofold = namedtuple("Twofold", ("value", "error"))

# (device, dtype, stream) -> workspace tensor, zeroed once (the kernel leaves it
# zeroed).  Keyed by stream: reductions on different streams may run concurrently
# and must not share the tile-partial array or the ticket counter.
_WS = {}
# Workspaces are never handed back to the allocator while a captured CUDA graph
# may still reference them: one outgrown by a larger reduction is retired here
# (kept alive) instead of freed, and a reduction captured into a graph gets a
# workspace of its own, so graph replays never share a ticket counter with eager
# reductions (or with another graph) and never write into recycled memory.
_WS_RETIRED = []
_WS_CAPTURED = []


def geometry(dtype=np.float64):
    """(V, W, K) of the canonical order for a plane dtype."""
    V, W, K = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    dt = _lib.TF_F64 if np.dtype(dtype) == np.float64 else _lib.TF_F32
    _lib.check(_lib.lib().tf_reduce_geometry(dt, ctypes.byref(V), ctypes.byref(W),
                                             ctypes.byref(K)), "geometry")
    return V.value, W.value, K.value


def tile_elems(dtype=np.float64) -> int:
    V, W, K = geometry(dtype)
    return V * W * K


def workspace(device: int, dtype_id: int, n: int, stream=None, factor: int = 1):
    need = factor * _lib.lib().tf_reduce_workspace_bytes(0, dtype_id, n)
    stream = stream if stream is not None else torch.cuda.current_stream(device)
    if torch.cuda.is_current_stream_capturing():
        with torch.cuda.stream(stream):  # allocated and zeroed inside the capture
            ws = torch.zeros(max(need, 4096), dtype=torch.uint8, device="cuda:%d" % device)
        _WS_CAPTURED.append(ws)
        return ws
    key = (device, dtype_id, stream.cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < need:
        with torch.cuda.stream(stream):  # allocated, zeroed and used on one stream
            new = torch.zeros(max(need, 4096), dtype=torch.uint8, device="cuda:%d" % device)
        if ws is not None:
            _WS_RETIRED.append(ws)
        ws = _WS[key] = new
    return ws


def _reduce(name, rop, ins, out=None):
    planes = [_describe(name, p) for p in ins]
    first = planes[0]
    for p in planes[1:]:
        if p.dtype != first.dtype:
            raise ValueError("%s: planes mix %s and %s" % (name, first.dtype, p.dtype))
        if p.n != first.n:
            raise ValueError("%s: plane lengths differ (%d vs %d)" % (name, first.n, p.n))
    if all(p.kind == "host" for p in planes):
        # numpy planes: pipelined through the device by tf_reduce_host, same bits
        if out is not None:
            raise ValueError("%s: out= is for CUDA planes" % name)
        dev = torch.cuda.current_device() if torch is not None else 0
        _lib.ensure_device(dev)
        from .kernels import _maybe_register

        for p in planes:
            if isinstance(p.obj, np.ndarray):
                _maybe_register(p.obj)
        dt = _dtype_id(first.dtype)
        res = np.zeros(2, first.dtype)
        rc = _lib.lib().tf_reduce_host(_lib.ROP_IDS[rop], dt, first.n, planes[0].ptr,
                                       planes[1].ptr if len(planes) > 1 else None,
                                       res.ctypes.data, dev)
        _lib.check(rc, name)
        return Twofold(float(res[0]), float(res[1]))
    if any(p.kind != "cuda" for p in planes):
        raise ValueError("%s: planes mix host arrays and CUDA tensors" % name)
    if len({p.device for p in planes}) != 1:
        raise ValueError("%s: planes live on different devices" % name)
    dev = first.device
    _lib.ensure_device(dev)
    dt = _dtype_id(first.dtype)
    tdt = torch.float64 if dt == _lib.TF_F64 else torch.float32
    res = out if out is not None else torch.empty(2, dtype=tdt, device="cuda:%d" % dev)
    if (res.dtype != tdt or not res.is_cuda or res.numel() < 2 or not res.is_contiguous()
            or res.get_device() != dev):
        raise ValueError("%s: out must be a contiguous 2-element CUDA tensor of the plane "
                         "dtype on the planes' device" % name)
    ws = workspace(dev, dt, first.n)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = _lib.lib().tf_reduce(_lib.ROP_IDS[rop], dt, first.n, planes[0].ptr,
                                  planes[1].ptr if len(planes) > 1 else None,
                                  res.data_ptr(), ws.data_ptr(), ws.numel(), stream)
    _lib.check(rc, name)
    if out is not None:
        return out
    v = res.cpu().tolist()
    return Twofold(v[0], v[1])


def vtsum(x, out=None):
    """Twofold sum of a plane: lanes fold ``_tadd1`` from (x, +0); trees of ``_tadd``."""
    return _reduce("vtsum", "sum", (x,), out)


def vtsum2(x, out=None):
    """Twofold sum of a TwofoldArray: lanes fold ``_tadd`` from (x0, x1)."""
    x0, x1 = x
    return _reduce("vtsum2", "sum2", (x0, x1), out)


def vtdot(x, y, out=None):
    """Twofold dot: lanes fold ``_tadd`` of ``_two_prod(x_i, y_i)``."""
    return _reduce("vtdot", "dot", (x, y), out)


def host_batch(calls, device=None):
    """Several reductions over host (numpy) planes in ONE pipelined pass.

    ``calls`` is a list of ``("vtsum", x)``, ``("vtsum2", (x0, x1))`` or
    ``("vtdot", x, y)``; all planes share one length and dtype.  Each distinct
    plane crosses the host link once however many reductions read it, so
    ``[("vtdot", x, y), ("vtsum", x)]`` moves x once.  Returns one ``Twofold`` per
    call, bit-identical to the calls made one by one (tf_reduce_host_batch).
    """
    if not calls:
        return []
    rops, a_ptrs, b_ptrs, first, seen = [], [], [], None, []
    for call in calls:
        name = call[0]
        if name == "vtsum":
            rop, ins = "sum", (call[1],)
        elif name == "vtsum2":
            rop, ins = "sum2", tuple(call[1])
        elif name == "vtdot":
            rop, ins = "dot", (call[1], call[2])
        else:
            raise ValueError("host_batch: unknown reduction %r" % (name,))
        planes = [_describe(name, p) for p in ins]
        seen.extend(planes)
        for p in planes:
            if p.kind != "host":
                raise ValueError("%s: host_batch takes numpy (host) planes" % name)
            if first is None:
                first = p
            elif p.dtype != first.dtype:
                raise ValueError("%s: planes mix %s and %s" % (name, first.dtype, p.dtype))
            elif p.n != first.n:
                raise ValueError("%s: plane lengths differ (%d vs %d)" % (name, first.n, p.n))
        rops.append(_lib.ROP_IDS[rop])
        a_ptrs.append(planes[0].ptr)
        b_ptrs.append(planes[1].ptr if len(planes) > 1 else None)
    from .kernels import _maybe_register

    for p in seen:
        if isinstance(p.obj, np.ndarray):
            _maybe_register(p.obj)
    dev = device if device is not None else (torch.cuda.current_device() if torch is not None else 0)
    _lib.ensure_device(dev)
    res = np.zeros((len(calls), 2), first.dtype)
    arr = (ctypes.c_int * len(rops))(*rops)
    rc = _lib.lib().tf_reduce_host_batch(len(rops), arr, _dtype_id(first.dtype), first.n,
                                         _lib.ptr_array(a_ptrs), _lib.ptr_array(b_ptrs),
                                         res.ctypes.data, dev)
    _lib.check(rc, "host_batch")
    return [Twofold(float(r[0]), float(r[1])) for r in res]


_RED_NAMES = {"vtsum": "sum", "vtsum2": "sum2", "vtdot": "dot"}


def _red_call(call):
    name = call[0]
    if name not in _RED_NAMES:
        raise ValueError("batch: unknown reduction %r" % (name,))
    ins = tuple(call[1]) if name == "vtsum2" else tuple(call[1:])
    if len(ins) != (1 if name == "vtsum" else 2):
        raise ValueError("%s: wrong number of planes" % name)
    return name, _RED_NAMES[name], ins


def batch(calls, out=None):
    """Several reductions over the same CUDA planes, two per pass.

    ``calls`` as for ``host_batch`` (numpy planes are routed there).  Two
    consecutive calls that read the same plane(s), e.g. ``[("vtdot", x, y),
    ("vtsum", x)]``, run as ONE kernel (tf_reduce_pair) that reads each plane
    once; any other call runs on its own.  Each result is bit-identical to its
    single reduction.  Returns a list of ``Twofold``, or with ``out`` (a
    (len(calls), 2) CUDA tensor) fills it asynchronously and returns it.
    """
    if not calls:
        return [] if out is None else out
    parsed = [_red_call(c) for c in calls]
    descs = [[_describe(name, p) for p in ins] for name, _, ins in parsed]
    kinds = {d.kind for ds in descs for d in ds}
    if kinds == {"host"}:
        if out is not None:
            raise ValueError("batch: out= is for CUDA planes")
        return host_batch(calls)
    if kinds != {"cuda"}:
        raise ValueError("batch: planes mix host arrays and CUDA tensors")
    first = descs[0][0]
    for (name, _, _), ds in zip(parsed, descs):
        for d in ds:
            if d.dtype != first.dtype or d.n != first.n or d.device != first.device:
                raise ValueError("%s: batch planes mix dtypes, lengths or devices" % name)
    dev, dt, n = first.device, _dtype_id(first.dtype), first.n
    _lib.ensure_device(dev)
    tdt = torch.float64 if dt == _lib.TF_F64 else torch.float32
    res = out if out is not None else torch.empty((len(calls), 2), dtype=tdt,
                                                  device="cuda:%d" % dev)
    if res.dtype != tdt or not res.is_cuda or tuple(res.shape) != (len(calls), 2) \
            or not res.is_contiguous():
        raise ValueError("batch: out must be a contiguous (len(calls), 2) CUDA tensor")
    L = _lib.lib()
    i = 0
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        while i < len(calls):
            a1 = descs[i]
            pair = None
            if i + 1 < len(calls):
                a2 = descs[i + 1]
                b = [ds[1].ptr for ds in (a1, a2) if len(ds) > 1]
                if a1[0].ptr == a2[0].ptr and len(set(b)) <= 1:
                    pair = b[0] if b else None
            if pair is not None or (i + 1 < len(calls) and a1[0].ptr == descs[i + 1][0].ptr
                                    and len(a1) == len(descs[i + 1]) == 1):
                ws = workspace(dev, dt, max(n, 1), stream, factor=2)
                rc = L.tf_reduce_pair(_lib.ROP_IDS[parsed[i][1]], _lib.ROP_IDS[parsed[i + 1][1]],
                                      dt, n, a1[0].ptr, pair, res[i].data_ptr(), ws.data_ptr(),
                                      ws.numel(), stream.cuda_stream)
                _lib.check(rc, "batch")
                i += 2
            else:
                name, rop, ins = parsed[i]
                _reduce(name, rop, ins, out=res[i])
                i += 1
    if out is not None:
        return out
    return [Twofold(v[0], v[1]) for v in res.cpu().tolist()]


def combine(partials, counts, out=None):
    """Adjacent-pair ``_tadd`` tree over per-shard partials (g x 2 CUDA tensor)."""
    p = partials.contiguous()
    g = p.shape[0]
    dt = _lib.TF_F64 if p.dtype == torch.float64 else _lib.TF_F32
    res = out if out is not None else torch.empty(2, dtype=p.dtype, device=p.device)
    c = (ctypes.c_int64 * max(g, 1))(*[int(v) for v in counts])
    with torch.cuda.device(p.device):
        stream = torch.cuda.current_stream(p.device).cuda_stream
        rc = _lib.lib().tf_combine(dt, g, p.data_ptr(), c, res.data_ptr(), stream)
    _lib.check(rc, "combine")
    if out is not None:
        return out
    v = res.cpu().tolist()
    return Twofold(v[0], v[1])


def vthorner(coeffs, x, out):
    """out = twofold Horner of Σ_k coeffs[k]·x^k (ascending powers) at every x_i."""
    c = [float(v) for v in coeffs]
    if not c:
        raise ValueError("vthorner: need at least one coefficient")
    r0, r1 = out
    planes = _check("vthorner", (x,), (r0, r1))
    first = planes[0]
    if first.n == 0:
        return
    carr = (ctypes.c_double * len(c))(*c)
    if first.kind == "host":  # numpy planes: through the host pipeline (tf_horner_host)
        dev = torch.cuda.current_device() if torch is not None else 0
        _lib.ensure_device(dev)
        rc = _lib.lib().tf_horner_host(_dtype_id(first.dtype), first.n, first.ptr, carr,
                                       len(c) - 1, planes[1].ptr, planes[2].ptr, dev)
        _lib.check(rc, "vthorner")
        return
    dev = first.device
    _lib.ensure_device(dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = _lib.lib().tf_horner(_dtype_id(first.dtype), first.n, first.ptr, carr, len(c) - 1,
                                  planes[1].ptr, planes[2].ptr, stream)
    _lib.check(rc, "vthorner")


def binomial_coeffs(degree=20):
    """Coefficients of the expanded (x-1)^degree, ascending powers (exact in f64)."""
    from math import comb

    return [float((-1) ** (degree - k) * comb(degree, k)) for k in range(degree + 1)]


__all__ = ["Twofold", "vtsum", "vtsum2", "vtdot", "vthorner", "combine", "host_batch", "batch",
           "geometry",
           "tile_elems", "binomial_coeffs", "TwofoldArray"]
