"""Elementwise twofold kernels on B200 — drop-in for ``twofold.kernels``.

Same surface as the reference module (/root/reference/pkg/src/twofold/kernels.py):
``TwofoldArray``, ``CoupledArray``, ``KernelSpec``, ``KERNELS`` (22 entries in
registry order, kernels.py:157-180), one module attribute per kernel
(``vtadd2`` ... ``vpdiv1``, kernels.py:242-247) and ``empty_twofold``
(kernels.py:250-255).  Signatures by arity (kernels.py:191-234):

    "22": f(x: TwofoldArray, y: TwofoldArray, out)     "u2": f(x: TwofoldArray, out)
    "21": f(x: TwofoldArray, y: plane, out)            "u1": f(x: plane, out)
    "11": f(x: plane, y: plane, out)

Planes are 1-D contiguous float32/float64 arrays:

* CUDA tensors (torch) — the B200 path: one asynchronous launch of the
  sm_100a kernel on the current torch stream (``tf_elementwise``);
* numpy arrays (or CPU tensors) — the reference's own calling convention: the
  library pipelines host->device copies, the kernel and device->host copies
  and returns when ``out`` holds the result (``tf_elementwise_host``).  This is
  the end-to-end path; there is no CPU arithmetic anywhere.

Contract kept from the reference (kernels.py:1-17, 123-147): callers allocate
every plane; every output index is written exactly once; arguments are validated
before anything is launched, raising ``ValueError("<kernel>: <reason>")`` with
the reference's message fragments; outputs may not alias inputs (even element-
aligned), inputs may alias each other; n == 0 is a no-op; numeric specials never
raise.  ``KernelSpec.loop`` is the raw launcher without validation (as used by
bench.py:256-262 in the reference).
"""

from __future__ import annotations

from collections import namedtuple

import numpy as np

from . import _lib

try:  # torch is the buffer manager for device planes; optional for host planes
    import torch
except Exception:  # pragma: no cover
    torch = None

TwofoldArray = namedtuple("TwofoldArray", ("value", "error"))
TwofoldArray.__doc__ = """Structure-of-arrays twofold: value and error planes."""


class CoupledArray(TwofoldArray):
    """A twofold array whose elements are non-overlapping pairs."""

    __slots__ = ()


KernelSpec = namedtuple(
    "KernelSpec",
    ("name", "arity", "core", "out_kind", "baseline", "scalar_name", "func", "loop"),
)
KernelSpec.__doc__ = """One kernel: its device launcher, core id and scalar twin.

arity as in the reference ("22", "21", "11", "u2", "u1"); ``core`` is the op id of
the device core in libtwofold_b200 (include/twofold_b200.h, enum tf_op);
baseline names the plain-arithmetic op the benchmark divides by; scalar_name is
the reference scalar operation the kernel matches bitwise.
"""

# name, arity, op id, out kind, baseline, scalar twin — kernels.py:157-180
_TABLE = [
    ("vtadd2", "22", 0, TwofoldArray, "add", "tadd"),
    ("vtsub2", "22", 1, TwofoldArray, "sub", "tsub"),
    ("vtmul2", "22", 2, TwofoldArray, "mul", "tmul"),
    ("vtdiv2", "22", 3, TwofoldArray, "div", "tdiv"),
    ("vtadd1", "21", 4, TwofoldArray, "add", "tadd1"),
    ("vtsub1", "21", 5, TwofoldArray, "sub", "tsub1"),
    ("vtmul1", "21", 6, TwofoldArray, "mul", "tmul1"),
    ("vtdiv1", "21", 7, TwofoldArray, "div", "tdiv1"),
    ("vtadd", "11", 8, CoupledArray, "add", "two_sum"),
    ("vtsub", "11", 9, CoupledArray, "sub", "two_diff"),
    ("vtmul", "11", 10, CoupledArray, "mul", "two_prod"),
    ("vtdiv", "11", 11, CoupledArray, "div", "tdiv0"),
    ("vtsqrt1", "u2", 12, TwofoldArray, "sqrt", "tsqrt"),
    ("vtsqrt", "u1", 13, CoupledArray, "sqrt", "tsqrt0"),
    ("vpadd2", "22", 14, CoupledArray, "add", "padd"),
    ("vpsub2", "22", 15, CoupledArray, "sub", "psub"),
    ("vpmul2", "22", 16, CoupledArray, "mul", "pmul_coupled"),
    ("vpdiv2", "22", 17, CoupledArray, "div", "pdiv_coupled"),
    ("vpadd1", "21", 18, CoupledArray, "add", "padd1"),
    ("vpsub1", "21", 19, CoupledArray, "sub", "psub1"),
    ("vpmul1", "21", 20, CoupledArray, "mul", "pmul1"),
    ("vpdiv1", "21", 21, CoupledArray, "div", "pdiv1"),
]

# raw exact-transform loops (not registry kernels), as test_acceptance.py:42-43
# drives _loop11(_div_rem) / _loop1u(_sqrt_resid)
RAW_OPS = {"div_rem": (22, 2), "sqrt_resid": (23, 1)}

_DOCS = {
    "22": "Elementwise ``%s`` of two twofold arrays into ``out``.",
    "21": "Elementwise ``%s`` of a twofold array and a scalar array into ``out``.",
    "11": "Elementwise ``%s`` of two scalar arrays into coupled ``out``.",
    "u2": "Elementwise ``%s`` of a twofold array into ``out``.",
    "u1": "Elementwise ``%s`` of a scalar array into coupled ``out``.",
}

_NP_DTYPES = (np.dtype(np.float32), np.dtype(np.float64))


# --------------------------------------------------------------------------
# plane introspection (numpy arrays, CPU tensors and CUDA tensors)


class _Plane:
    __slots__ = ("obj", "kind", "dtype", "n", "ptr", "nbytes", "device")

    def __init__(self, obj, kind, dtype, n, ptr, nbytes, device):
        self.obj, self.kind, self.dtype, self.n = obj, kind, dtype, n
        self.ptr, self.nbytes, self.device = ptr, nbytes, device


def _is_tensor(a) -> bool:
    return torch is not None and isinstance(a, torch.Tensor)


_F64, _F32 = np.dtype(np.float64), np.dtype(np.float32)
_TORCH_DT = {}
if torch is not None:
    _TORCH_DT = {torch.float64: _F64, torch.float32: _F32}
    _Tensor = torch.Tensor
else:  # pragma: no cover
    _Tensor = ()


def _describe(name, a) -> _Plane:
    if isinstance(a, _Tensor):  # the hot path: one call per plane per launch
        dt = _TORCH_DT.get(a.dtype)
        if a.dim() != 1 or not a.is_contiguous():
            raise ValueError("%s: planes must be 1-D and contiguous" % name)
        if dt is None:
            raise ValueError("%s: planes must be float32 or float64, got %s" % (name, a.dtype))
        dev = a.get_device()
        if dev >= 0:
            return _Plane(a, "cuda", dt, a.shape[0], a.data_ptr(), a.nbytes, dev)
        return _Plane(a, "host", dt, a.shape[0], a.data_ptr(), a.nbytes, None)
    if isinstance(a, np.ndarray):
        if a.ndim != 1 or not a.flags.c_contiguous:
            raise ValueError("%s: planes must be 1-D and contiguous" % name)
        if a.dtype not in _NP_DTYPES:
            raise ValueError("%s: planes must be float32 or float64, got %s" % (name, a.dtype))
        return _Plane(a, "host", a.dtype, a.shape[0], a.ctypes.data, a.nbytes, None)
    raise ValueError("%s: planes must be numpy arrays or CUDA tensors, got %r"
                     % (name, type(a).__name__))


def _overlap(p: _Plane, q: _Plane) -> bool:
    if p.kind != q.kind or p.nbytes == 0 or q.nbytes == 0:
        return False
    if p.kind == "cuda" and p.device != q.device:
        return False
    return p.ptr < q.ptr + q.nbytes and q.ptr < p.ptr + p.nbytes


def _check(name, ins, outs):
    """Validate before any launch (kernels.py:123-147); returns described planes."""
    planes = [_describe(name, a) for a in tuple(ins) + tuple(outs)]
    first = planes[0]
    for p in planes[1:]:
        if p.dtype != first.dtype:
            raise ValueError("%s: planes mix %s and %s" % (name, first.dtype, p.dtype))
        if p.n != first.n:
            raise ValueError("%s: plane lengths differ (%d vs %d)" % (name, first.n, p.n))
    kinds = {p.kind for p in planes}
    if len(kinds) != 1:
        raise ValueError("%s: planes mix host arrays and CUDA tensors" % name)
    if first.kind == "cuda" and len({p.device for p in planes}) != 1:
        raise ValueError("%s: planes live on different devices" % name)
    pin, pout = planes[: len(ins)], planes[len(ins):]
    for o in pout:
        # the reference's numba loop refuses a read-only out array at call time;
        # here the library would write through the pointer, so refuse up front
        if isinstance(o.obj, np.ndarray) and not o.obj.flags.writeable:
            raise ValueError("%s: out planes must be writeable" % name)
    for o in pout:
        for a in pin:
            if _overlap(o, a):
                raise ValueError("%s: out must not alias an input" % name)
    if _overlap(pout[0], pout[1]):
        raise ValueError("%s: out planes overlap each other" % name)
    return planes


# --------------------------------------------------------------------------
# launchers


def _dtype_id(dt) -> int:
    return _lib.TF_F64 if dt == np.dtype(np.float64) else _lib.TF_F32


def _raw_stream(dev):
    """cudaStream_t of torch's current stream on `dev` (no Stream object)."""
    try:
        return torch._C._cuda_getCurrentRawStream(dev)
    except AttributeError:  # pragma: no cover - older torch
        return torch.cuda.current_stream(dev).cuda_stream


def _launch(name, op, planes, nin):
    """Raw launch over described planes (device: async; host: synchronous)."""
    L = _lib._lib or _lib.lib()
    first = planes[0]
    n = first.n
    if n == 0:
        return
    ins = _lib.ptr_array([p.ptr for p in planes[:nin]])
    outs = _lib.ptr_array([p.ptr for p in planes[nin:]])
    if first.kind == "cuda":
        dev = first.device
        if dev not in _lib._selftested:
            _lib.ensure_device(dev)
        stream = _raw_stream(dev)
        if torch.cuda.current_device() == dev:
            rc = L.tf_elementwise(op, _dtype_id(first.dtype), n, ins, outs, stream)
        else:
            with torch.cuda.device(dev):
                rc = L.tf_elementwise(op, _dtype_id(first.dtype), n, ins, outs, stream)
        if rc:
            _lib.check(rc, name)
    else:
        dev = torch.cuda.current_device() if torch is not None else 0
        _lib.ensure_device(dev)
        for p in planes:
            if isinstance(p.obj, np.ndarray):
                _maybe_register(p.obj)
        rc = L.tf_elementwise_host(op, _dtype_id(first.dtype), n, ins, outs, dev)
        _lib.check(rc, name)


def _make_loop(name, op, nin):
    def loop(*planes):
        """Raw launcher: no validation beyond the library's own (spec.loop)."""
        desc = [_describe(name, p) for p in planes]
        _launch(name, op, desc, nin)

    loop.__name__ = name + "_loop"
    return loop


def _build(name, arity, op, out_kind, baseline, scalar_name):
    nin = {"22": 4, "21": 3, "11": 2, "u2": 2, "u1": 1}[arity]
    loop = _make_loop(name, op, nin)

    if arity == "22":
        def kern(x, y, out):
            x0, x1 = x
            y0, y1 = y
            r0, r1 = out
            _launch(name, op, _check(name, (x0, x1, y0, y1), (r0, r1)), 4)
    elif arity == "21":
        def kern(x, y, out):
            x0, x1 = x
            r0, r1 = out
            _launch(name, op, _check(name, (x0, x1, y), (r0, r1)), 3)
    elif arity == "11":
        def kern(x, y, out):
            r0, r1 = out
            _launch(name, op, _check(name, (x, y), (r0, r1)), 2)
    elif arity == "u2":
        def kern(x, out):
            x0, x1 = x
            r0, r1 = out
            _launch(name, op, _check(name, (x0, x1), (r0, r1)), 2)
    else:
        def kern(x, out):
            r0, r1 = out
            _launch(name, op, _check(name, (x,), (r0, r1)), 1)

    kern.__name__ = name
    kern.__qualname__ = name
    kern.__doc__ = _DOCS[arity] % scalar_name
    return KernelSpec(name, arity, op, out_kind, baseline, scalar_name, kern, loop)


KERNELS = {}
for _row in _TABLE:
    _spec = _build(*_row)
    KERNELS[_spec.name] = _spec
    globals()[_spec.name] = _spec.func
del _row, _spec


def raw_loop(name):
    """Launcher for the raw exact transforms div_rem / sqrt_resid (no validation)."""
    op, nin = RAW_OPS[name]
    return _make_loop(name, op, nin)


def _torch_dtype(dt):
    if torch is not None and isinstance(dt, torch.dtype):
        if dt in (torch.float32, torch.float64):
            return dt
        raise ValueError("dtype must be float32 or float64, got %s" % dt)
    d = np.dtype(dt)
    if d not in _NP_DTYPES:
        raise ValueError("dtype must be float32 or float64, got %s" % d)
    return d


def empty_twofold(n, dtype=np.float64, kind=TwofoldArray, device=None, pin_memory=False):
    """Allocate an uninitialized twofold array of n elements (kernels.py:250-255).

    The reference's default is kept: a numpy dtype (the default float64) with no
    ``device`` gives numpy planes, exactly as ``twofold.kernels.empty_twofold``
    (optionally page-locked with ``pin_memory=True``, the fast host path).  CUDA
    planes are opt-in: a torch dtype (``torch.float64``) allocates on the
    current CUDA device, and ``device="cuda"`` / ``"cuda:k"`` / an index picks
    one explicitly; ``device="cpu"`` forces numpy planes.
    """
    dt = _torch_dtype(dtype)
    is_torch_dt = torch is not None and isinstance(dt, torch.dtype)
    if is_torch_dt:
        tdt = dt
    else:
        tdt = None
        if torch is not None:
            tdt = torch.float64 if dt == np.dtype(np.float64) else torch.float32
    if device is None:
        device = "cuda" if is_torch_dt else "cpu"
    if device in ("cpu", "host"):
        if pin_memory and torch is not None:
            planes = [torch.empty(n, dtype=tdt, pin_memory=True).numpy() for _ in range(2)]
            return kind(*planes)
        npdt = dt if not (torch is not None and isinstance(dt, torch.dtype)) else (
            np.float64 if dt == torch.float64 else np.float32)
        return kind(np.empty(n, npdt), np.empty(n, npdt))
    if torch is None:
        raise RuntimeError("empty_twofold: torch is required for device planes")
    dev = torch.device(device if not isinstance(device, int) else "cuda:%d" % device)
    return kind(torch.empty(n, dtype=tdt, device=dev), torch.empty(n, dtype=tdt, device=dev))


__all__ = ["TwofoldArray", "CoupledArray", "KernelSpec", "KERNELS",
           "empty_twofold"] + [row[0] for row in _TABLE]


def _parse_batch(calls, who):
    """Validate a batch of ``(name, *args, out)`` calls (each with its kernel's own
    signature); returns (op ids, input pointers (4 per op), output pointers (2 per
    op), the first plane's description, every description)."""
    ops, ins, outs, first, descs = [], [], [], None, []
    for call in calls:
        name, args = call[0], call[1:]
        spec = KERNELS[name]
        if spec.arity in ("22",):
            (x0, x1), (y0, y1), (r0, r1) = args
            planes = (x0, x1, y0, y1)
        elif spec.arity == "21":
            (x0, x1), y, (r0, r1) = args
            planes = (x0, x1, y)
        elif spec.arity == "11":
            x, y, (r0, r1) = args
            planes = (x, y)
        elif spec.arity == "u2":
            (x0, x1), (r0, r1) = args
            planes = (x0, x1)
        else:
            x, (r0, r1) = args
            planes = (x,)
        desc = _check(name, planes, (r0, r1))
        if first is None:
            first = desc[0]
        elif (desc[0].dtype != first.dtype or desc[0].n != first.n
              or desc[0].kind != first.kind or desc[0].device != first.device):
            raise ValueError("%s: batch planes mix dtypes, lengths or devices" % name)
        ops.append(spec.core)
        ins.extend([d.ptr for d in desc[:len(planes)]] + [None] * (4 - len(planes)))
        outs.extend([d.ptr for d in desc[len(planes):]])
        descs.extend(desc)
    return ops, ins, outs, first, descs


def host_batch(calls, device=None):
    """Run several kernels on host (numpy) planes in ONE pipelined pass.

    ``calls`` is a list of ``(name, *args, out)`` tuples with each kernel's own
    signature, e.g. ``[("vtadd2", x, y, o1), ("vtsqrt1", x, o2)]``.  All planes
    share one length and dtype.  Each distinct input plane crosses the host link
    once per chunk however many calls read it; outputs come back in call order,
    so the results equal running the calls one by one.  No output may overlap
    any input of the batch (an intra-batch dependency), checked before any copy.
    """
    import ctypes

    if not calls:
        return
    ops, ins, outs, first, descs = _parse_batch(calls, "host_batch")
    if any(d.kind != "host" for d in descs):
        raise ValueError("%s: host_batch takes numpy (host) planes" % calls[0][0])
    for d in descs:
        if isinstance(d.obj, np.ndarray):
            _maybe_register(d.obj)
    # cross-call aliasing (an output of one call over an input of another) is
    # rejected by the library before any copy (TF_EINVAL -> ValueError)
    L = _lib.lib()
    dev = device if device is not None else (torch.cuda.current_device() if torch is not None else 0)
    _lib.ensure_device(dev)
    arr_ops = (ctypes.c_int * len(ops))(*ops)
    rc = L.tf_elementwise_host_batch(len(ops), arr_ops, _dtype_id(first.dtype), first.n,
                                     _lib.ptr_array(ins), _lib.ptr_array(outs), dev)
    _lib.check(rc, "host_batch")


BATCH_MAX = 8  # ops per device launch (tf_elementwise_batch)


def batch(calls):
    """Run several kernels over the same planes as ONE device launch per 8 calls.

    ``calls`` as for ``host_batch``.  CUDA-tensor planes: ``tf_elementwise_batch``
    on the current stream; each distinct input plane is read from HBM once,
    every call's output is written once, and the results equal running the calls
    one by one (bit for bit).  Host (numpy) planes go to ``host_batch``.  No
    output may overlap any input of the batch (ValueError before any launch).
    """
    import ctypes

    if not calls:
        return
    ops, ins, outs, first, descs = _parse_batch(calls, "batch")
    if first.kind != "cuda":
        return host_batch(calls)
    # every group's outputs against every input of the whole batch
    span = first.n * first.dtype.itemsize
    in_ptrs = [p for p in ins if p is not None]
    for o in outs:
        if first.n and any(o < q + span and q < o + span for q in in_ptrs):
            raise ValueError("batch: out must not alias an input")
    L = _lib.lib()
    _lib.ensure_device(first.device)
    with torch.cuda.device(first.device):
        stream = torch.cuda.current_stream().cuda_stream
        for g in range(0, len(ops), BATCH_MAX):
            k = min(BATCH_MAX, len(ops) - g)
            arr_ops = (ctypes.c_int * k)(*ops[g:g + k])
            rc = L.tf_elementwise_batch(k, arr_ops, _dtype_id(first.dtype), first.n,
                                        _lib.ptr_array(ins[4 * g:4 * (g + k)]),
                                        _lib.ptr_array(outs[2 * g:2 * (g + k)]), stream)
            _lib.check(rc, "batch")


# --------------------------------------------------------------------------
# page-locking of reused pageable numpy planes (host path)
#
# A pageable plane goes through pinned staging (three trips through host DRAM).
# A plane seen TF_HOST_REGISTER_AFTER (4) times — the reference's loops reuse
# their arrays — is page-locked in place with tf_host_register, within a byte
# budget (LRU), and unregistered by a weakref finalizer before numpy releases
# its memory.

import collections as _collections
import os as _os
import threading as _threading
import weakref as _weakref

_REG_LOCK = _threading.Lock()
_REG = _collections.OrderedDict()  # owner address -> (nbytes, finalizer)
# owner address -> (uses, weakref to the owner).  The weakref ties a count to the
# array that earned it (a new array at a recycled address starts from zero) and
# lets dead entries be pruned; the table is capped at _SEEN_MAX live entries.
_SEEN = _collections.OrderedDict()
_SEEN_MAX = 256
_REG_MIN = 32 << 20
_REG_BUDGET = int(float(_os.environ.get("TF_HOST_REGISTER_GB", "16")) * (1 << 30))
# page-locking costs ~80 ms per GiB (measured) and saves ~40% of a staged call,
# so it pays for itself only on planes reused several times
_REG_AFTER = int(_os.environ.get("TF_HOST_REGISTER_AFTER", "4"))


def _owner(a):
    o = a
    while isinstance(o, np.ndarray) and o.base is not None:
        o = o.base
    if not isinstance(o, np.ndarray) or not o.flags.owndata:
        return None  # memory owned elsewhere (torch pinned, mmap, ...): leave it alone
    return o


def _unregister(addr):
    try:
        (_lib._lib or _lib.lib()).tf_host_unregister(addr)
    except Exception:  # pragma: no cover - interpreter shutdown
        pass
    with _REG_LOCK:
        _REG.pop(addr, None)


def _maybe_register(a):
    if _REG_BUDGET <= 0:
        return
    o = _owner(a)
    if o is None or o.nbytes < _REG_MIN:
        return
    addr = o.ctypes.data
    with _REG_LOCK:
        if addr in _REG:
            _REG.move_to_end(addr)
            return
        uses, ref = _SEEN.pop(addr, (0, None))
        if ref is None or ref() is not o:
            uses = 0  # first sight, or a new array at a recycled address
        uses += 1
        _SEEN[addr] = (uses, _weakref.ref(o))
        if len(_SEEN) > _SEEN_MAX:
            for k in [k for k, (_, r) in _SEEN.items() if r() is None]:
                del _SEEN[k]
            while len(_SEEN) > _SEEN_MAX:
                _SEEN.popitem(last=False)
        if uses < _REG_AFTER or o.nbytes > _REG_BUDGET:
            return
        total = sum(v[0] for v in _REG.values())
        while _REG and total + o.nbytes > _REG_BUDGET:
            old, (nb, fin) = _REG.popitem(last=False)
            fin.detach()
            (_lib._lib or _lib.lib()).tf_host_unregister(old)
            total -= nb
        if (_lib._lib or _lib.lib()).tf_host_register(addr, o.nbytes) != 0:
            _SEEN[addr] = (-(1 << 30), _weakref.ref(o))  # not registrable: stay staged
            return
        _REG[addr] = (o.nbytes, _weakref.finalize(o, _unregister, addr))
        _SEEN.pop(addr, None)
