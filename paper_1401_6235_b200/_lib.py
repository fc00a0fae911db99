"""ctypes binding of libtwofold_b200.so (include/twofold_b200.h).

The shared library is built in-tree (``python -m paper_1401_6235_b200.build`` or
``__graft_entry__.build()``) and loaded from ``paper_1401_6235_b200/_lib/``.
There is no fallback: if the library is missing or its device self-test fails,
every entry point raises.  ctypes releases the GIL for the duration of each call.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("TF_LIB_PATH") or
                (Path(__file__).resolve().parent / "_lib" / "libtwofold_b200.so"))

TF_OK, TF_EINVAL, TF_ECUDA, TF_ENOMEM, TF_ESELFTEST = 0, -1, -2, -3, -4
TF_F32, TF_F64 = 0, 1
ROP_IDS = {"sum": 0, "sum2": 1, "dot": 2}

_lock = threading.RLock()
_lib = None
_selftested = set()


class LibraryMissing(RuntimeError):
    pass


def _bind(L: ctypes.CDLL) -> None:
    vp, i64, ci, cd = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    pvp = ctypes.POINTER(vp)
    sig = {
        "tf_abi_version": (ci, []),
        "tf_last_error": (ctypes.c_char_p, []),
        "tf_num_inputs": (ci, [ci]),
        "tf_selftest": (ci, [ci]),
        "tf_elementwise": (ci, [ci, ci, i64, pvp, pvp, vp]),
        "tf_elementwise_host": (ci, [ci, ci, i64, pvp, pvp, ci]),
        "tf_host_register": (ci, [vp, ctypes.c_size_t]),
        "tf_host_unregister": (ci, [vp]),
        "tf_elementwise_host_batch": (ci, [ci, ctypes.POINTER(ci), ci, i64, pvp, pvp, ci]),
        "tf_elementwise_batch": (ci, [ci, ctypes.POINTER(ci), ci, i64, pvp, pvp, vp]),
        "tf_elementwise_il": (ci, [ci, ci, i64, vp, vp, vp, vp]),
        "tf_fused": (ci, [ci, ci, i64, pvp, pvp, vp]),
        "tf_interleave": (ci, [ci, i64, vp, vp, vp, vp]),
        "tf_deinterleave": (ci, [ci, i64, vp, vp, vp, vp]),
        "tf_reduce_geometry": (ci, [ci, ctypes.POINTER(ci), ctypes.POINTER(ci), ctypes.POINTER(ci)]),
        "tf_reduce_workspace_bytes": (ctypes.c_size_t, [ci, ci, i64]),
        "tf_reduce": (ci, [ci, ci, i64, vp, vp, vp, vp, ctypes.c_size_t, vp]),
        "tf_reduce_pair": (ci, [ci, ci, ci, i64, vp, vp, vp, vp, ctypes.c_size_t, vp]),
        "tf_combine": (ci, [ci, ci, vp, ctypes.POINTER(i64), vp, vp]),
        "tf_reduce_host": (ci, [ci, ci, i64, vp, vp, vp, ci]),
        "tf_reduce_host_batch": (ci, [ci, ctypes.POINTER(ci), ci, i64, vp, vp, vp, ci]),
        "tf_xgpu_mailbox": (ci, [ci, vp]),
        "tf_xgpu_open": (ci, [ci, ci, ci, vp]),
        "tf_xgpu_combine": (ci, [ci, vp, ctypes.POINTER(i64), vp]),
        "tf_xgpu_status": (ci, [ci]),
        "tf_xgpu_emulate": (ci, [ci, ci, vp, ctypes.POINTER(i64), ci, vp]),
        "tf_xgpu_reduce": (ci, [ci, ci, i64, vp, vp, vp, vp, ctypes.c_size_t,
                                ctypes.POINTER(i64), vp]),
        "tf_xgpu_reduce_emulate": (ci, [ci, ci, ci, vp, vp, ctypes.POINTER(i64), vp, vp]),
        "tf_xgpu_publish": (ci, [ci, vp, ctypes.POINTER(i64), vp]),
        "tf_xgpu_reduce_publish": (ci, [ci, ci, i64, vp, vp, vp, vp, ctypes.c_size_t,
                                        ctypes.POINTER(i64), vp]),
        "tf_xgpu_collect": (ci, [ci, vp, vp]),
        "tf_horner": (ci, [ci, i64, vp, ctypes.POINTER(cd), ci, vp, vp, vp]),
        "tf_horner_host": (ci, [ci, i64, vp, ctypes.POINTER(cd), ci, vp, vp, ci]),
        "tf_fill": (ci, [ci, ci, i64, ctypes.c_uint64, i64, cd, cd, vp, vp, vp]),
        "tf_dotted": (ci, [ci, ci, i64, vp, vp, vp, vp]),
        "tf_fp64_peak": (ci, [ci, ctypes.POINTER(cd), ctypes.POINTER(cd)]),
        "tf_fastpath_check": (ci, [ci, i64, ctypes.c_uint64, ctypes.POINTER(i64)]),
        "tf_gen_dot_host": (ci, [i64, cd, ctypes.c_uint64, vp, vp]),
        "tf_gen_ill": (ci, [ci, i64, i64, i64, cd, ctypes.c_uint64, ci, ci, vp, vp, vp]),
        "tf_gen_ill_host": (ci, [ci, i64, i64, i64, cd, ctypes.c_uint64, ci, ci, vp, vp, ci]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


EXPORTS = (
    "tf_abi_version", "tf_last_error", "tf_num_inputs", "tf_selftest", "tf_elementwise",
    "tf_elementwise_host", "tf_elementwise_host_batch", "tf_elementwise_batch", "tf_host_register", "tf_host_unregister", "tf_elementwise_il", "tf_fused", "tf_interleave", "tf_deinterleave",
    "tf_reduce_geometry", "tf_reduce_workspace_bytes", "tf_reduce", "tf_reduce_pair",
    "tf_combine", "tf_reduce_host", "tf_reduce_host_batch", "tf_xgpu_mailbox", "tf_xgpu_open", "tf_xgpu_combine",
    "tf_xgpu_status", "tf_xgpu_emulate", "tf_xgpu_reduce", "tf_xgpu_reduce_emulate",
    "tf_xgpu_publish", "tf_xgpu_reduce_publish", "tf_xgpu_collect", "tf_horner", "tf_horner_host", "tf_fill", "tf_dotted", "tf_fp64_peak", "tf_fastpath_check", "tf_gen_dot_host",
    "tf_gen_ill", "tf_gen_ill_host",
)


def lib() -> ctypes.CDLL:
    """Load (once) and return the library; raises LibraryMissing if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise LibraryMissing(
                    "libtwofold_b200.so not built (%s); run __graft_entry__.build()" % LIB_PATH)
            L = ctypes.CDLL(str(LIB_PATH))
            _bind(L)
            if L.tf_abi_version() != 1:
                raise LibraryMissing("libtwofold_b200.so ABI mismatch")
            _lib = L
    return _lib


def last_error() -> str:
    return lib().tf_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Map a status code to the reference's exception types."""
    if rc == TF_OK:
        return
    msg = last_error()
    if rc == TF_EINVAL:
        raise ValueError("%s: %s" % (what, msg))
    raise RuntimeError("%s failed (%d): %s" % (what, rc, msg))


def ensure_device(device: int) -> None:
    """Run the device self-test (the _fused_or_die analogue) once per device."""
    if device in _selftested:
        return
    L = lib()
    with _lock:
        if device in _selftested:
            return
        rc = L.tf_selftest(int(device))
        if rc != TF_OK:
            raise RuntimeError("twofold device self-test failed on cuda:%d: %s"
                               % (device, last_error()))
        _selftested.add(device)


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * max(len(ptrs), 1))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
