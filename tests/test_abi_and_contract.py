"""CPU-only checks: the C ABI library loads and exports every declared symbol;
the drop-in registry has the reference's shape; argument validation rejects
bad calls before anything is launched (kernels.py:123-147 contract, with the
reference's message fragments, test_kernels.py:182-257)."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol():
    from paper_1401_6235_b200 import _lib

    L = _lib.lib()
    header = (ROOT / "include" / "twofold_b200.h").read_text()
    declared = set(re.findall(r"\b(tf_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(_lib.EXPORTS)
    assert L.tf_abi_version() == 1


def test_num_inputs_and_geometry_without_gpu():
    import ctypes

    from paper_1401_6235_b200 import _lib

    L = _lib.lib()
    assert [L.tf_num_inputs(i) for i in range(24)] == [4, 4, 4, 4, 3, 3, 3, 3, 2, 2, 2, 2, 2, 1,
                                                      4, 4, 4, 4, 3, 3, 3, 3, 2, 1]
    assert L.tf_num_inputs(24) < 0 and "unknown op" in _lib.last_error()
    V, W, K = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert L.tf_reduce_geometry(1, ctypes.byref(V), ctypes.byref(W), ctypes.byref(K)) == 0
    assert (V.value, W.value, K.value) == (2, 256, 128)
    assert L.tf_reduce_workspace_bytes(0, 1, 1 << 30) == 256 + 16 * (1 << 14)


def test_gen_dot_host_is_deterministic(oracle):
    from paper_1401_6235_b200 import _lib

    n = 1 << 14
    xs = []
    for _ in range(2):
        x, y = np.empty(n), np.empty(n)
        assert _lib.lib().tf_gen_dot_host(n, 1e16, 3, x.ctypes.data, y.ctypes.data) == 0
        xs.append((x, y))
    assert np.array_equal(xs[0][0], xs[1][0]) and np.array_equal(xs[0][1], xs[1][1])
    s, t = oracle.exact("dot", *xs[0])
    cond = float(2 * t / abs(s))
    assert 0.5e16 < cond < 2e16, cond  # calibrated: the requested condition number


def test_registry_contents():
    from paper_1401_6235_b200 import kernels as K

    assert len(K.KERNELS) == 22
    hist = {}
    for spec in K.KERNELS.values():
        hist[spec.arity] = hist.get(spec.arity, 0) + 1
        assert spec.baseline in {"add", "sub", "mul", "div", "sqrt"}
        assert getattr(K, spec.name) is spec.func
    assert hist == {"22": 8, "21": 8, "11": 4, "u2": 1, "u1": 1}
    assert list(K.KERNELS) == ["vtadd2", "vtsub2", "vtmul2", "vtdiv2", "vtadd1", "vtsub1",
                               "vtmul1", "vtdiv1", "vtadd", "vtsub", "vtmul", "vtdiv",
                               "vtsqrt1", "vtsqrt", "vpadd2", "vpsub2", "vpmul2", "vpdiv2",
                               "vpadd1", "vpsub1", "vpmul1", "vpdiv1"]
    assert [s.core for s in K.KERNELS.values()] == list(range(22))


def test_out_kinds():
    from paper_1401_6235_b200 import kernels as K

    assert K.KERNELS["vtadd2"].out_kind is K.TwofoldArray
    assert K.KERNELS["vtadd"].out_kind is K.CoupledArray
    assert K.KERNELS["vpadd2"].out_kind is K.CoupledArray
    assert K.KERNELS["vtsqrt"].out_kind is K.CoupledArray
    assert K.KERNELS["vtsqrt1"].out_kind is K.TwofoldArray


def _planes(rng, n):
    v = rng.uniform(1, 2, n) * np.exp2(rng.integers(-3, 4, n)) * rng.choice([-1.0, 1.0], n)
    return v, v * 2.0**-52 * rng.uniform(-1, 1, n)


def _fresh(n=8, dtype=np.float64):
    from paper_1401_6235_b200 import kernels as K

    rng = np.random.default_rng(3)
    x = K.TwofoldArray(*[p.astype(dtype) for p in _planes(rng, n)])
    y = K.TwofoldArray(*[p.astype(dtype) for p in _planes(rng, n)])
    out = K.TwofoldArray(np.full(n, 7.0, dtype), np.full(n, 7.0, dtype))
    return x, y, out


def _rejected(fn, out, frag):
    with pytest.raises(ValueError, match=frag):
        fn()
    assert np.all(out.value == 7.0) and np.all(out.error == 7.0)


def test_rejections_happen_before_any_launch():
    # no GPU here: a call that got past validation would fail to launch, so a
    # ValueError with the right fragment proves validation came first
    from paper_1401_6235_b200 import kernels as K

    x, y, out = _fresh()
    short = K.TwofoldArray(y.value[:4].copy(), y.error[:4].copy())
    _rejected(lambda: K.vtadd2(x, short, out), out, "lengths differ")
    y32 = K.TwofoldArray(y.value.astype(np.float32), y.error.astype(np.float32))
    _rejected(lambda: K.vtadd2(x, y32, out), out, "mix")
    x16, _, _ = _fresh(16)
    _rejected(lambda: K.vtadd2(K.TwofoldArray(x16.value[::2], x16.error[::2]),
                               K.TwofoldArray(x16.value[::2], x16.error[::2]), out),
              out, "contiguous")
    _rejected(lambda: K.vtadd2(x, K.TwofoldArray(np.arange(8), np.arange(8)), out), out,
              "float32 or float64")
    _rejected(lambda: K.vtadd2(x, K.TwofoldArray(list(x.value), list(x.error)), out), out,
              "numpy arrays")
    _rejected(lambda: K.vtadd2(x, K.TwofoldArray(np.ones((2, 4)), np.ones((2, 4))), out), out,
              "1-D")
    with pytest.raises(ValueError, match="alias"):
        K.vtadd2(x, y, K.TwofoldArray(x.value, out.error))
    with pytest.raises(ValueError, match="alias"):
        K.vtadd2(x, y, K.TwofoldArray(out.value, y.error))
    same = np.full(8, 7.0)
    with pytest.raises(ValueError, match="overlap"):
        K.vtadd2(x, y, K.TwofoldArray(same, same))


def test_read_only_out_is_rejected():
    # a read-only numpy out plane (np.frombuffer over bytes, a read-only mmap)
    # is refused before anything is written through its pointer
    from paper_1401_6235_b200 import kernels as K

    x, y, out = _fresh()
    ro = np.frombuffer(bytes(8 * 8), dtype=np.float64)
    with pytest.raises(ValueError, match="writeable"):
        K.vtadd2(x, y, K.TwofoldArray(ro, out.error))
    assert np.all(ro == 0) and np.all(out.error == 7.0)
    # read-only INPUTS are fine (the reference reads them too)
    assert not ro.flags.writeable


def test_partial_overlap_is_aliasing():
    from paper_1401_6235_b200 import kernels as K

    buf = np.zeros(16)
    x = K.TwofoldArray(buf[0:8], buf[0:8])
    with pytest.raises(ValueError, match="alias"):
        K.vtadd2(x, x, K.TwofoldArray(buf[7:15], np.zeros(8)))


def test_validation_covers_every_arity():
    from paper_1401_6235_b200 import kernels as K

    n = 8
    rng = np.random.default_rng(5)
    for name, spec in K.KERNELS.items():
        v, e = _planes(rng, n)
        args = {"22": (K.TwofoldArray(v, e), K.TwofoldArray(v, e)),
                "21": (K.TwofoldArray(v, e), v), "11": (v, e),
                "u2": (K.TwofoldArray(np.abs(v), e),), "u1": (np.abs(v),)}[spec.arity]
        out = K.TwofoldArray(np.full(n - 1, 7.0), np.full(n - 1, 7.0))
        with pytest.raises(ValueError, match=name):
            spec.func(*args, out)
        assert np.all(out.value == 7.0)


def test_empty_twofold_host_and_errors():
    from paper_1401_6235_b200 import kernels as K

    z = K.empty_twofold(5, device="cpu")
    assert type(z) is K.TwofoldArray
    assert z.value.dtype == np.float64 and z.value.shape == (5,)
    z = K.empty_twofold(5, np.float32, K.CoupledArray, device="cpu")
    assert type(z) is K.CoupledArray and z.error.dtype == np.float32
    with pytest.raises(ValueError, match="float32 or float64"):
        K.empty_twofold(5, np.int32)


def test_empty_twofold_defaults_to_numpy_like_the_reference():
    # reference kernels.py:250-255: numpy planes; test_kernels.py:260-267 asserts
    # the np.dtype of each plane.  CUDA planes are opt-in (a torch dtype or device=)
    import torch

    from paper_1401_6235_b200 import kernels as K

    z = K.empty_twofold(5)
    assert type(z) is K.TwofoldArray and isinstance(z.value, np.ndarray)
    assert z.value.dtype == np.dtype(np.float64) and z.value.shape == (5,)
    z = K.empty_twofold(5, np.float32, K.CoupledArray)
    assert type(z) is K.CoupledArray and isinstance(z.error, np.ndarray)
    assert z.error.dtype == np.dtype(np.float32)
    # a torch dtype with device="cpu" still gives numpy planes of that width
    z = K.empty_twofold(3, torch.float32, device="cpu")
    assert isinstance(z.value, np.ndarray) and z.value.dtype == np.float32


def test_seen_table_is_bounded_and_tied_to_the_array(monkeypatch):
    # the reuse counter behind page-locking (kernels._maybe_register) keeps at
    # most _SEEN_MAX entries, and a new array at a recycled address starts at 0
    from paper_1401_6235_b200 import kernels as K

    monkeypatch.setattr(K, "_REG_MIN", 0)
    monkeypatch.setattr(K, "_REG_AFTER", 1 << 30)  # never actually page-lock here
    monkeypatch.setattr(K, "_SEEN", K._collections.OrderedDict())
    keep = [np.empty(4) for _ in range(3 * K._SEEN_MAX)]
    for a in keep:
        K._maybe_register(a)
    assert len(K._SEEN) <= K._SEEN_MAX
    a = np.empty(8)
    for _ in range(3):
        K._maybe_register(a)
    assert K._SEEN[a.ctypes.data][0] == 3
    addr = a.ctypes.data
    del a
    b = np.empty(8)
    K._maybe_register(b)
    if b.ctypes.data == addr:  # recycled address: the old count does not carry over
        assert K._SEEN[addr][0] == 1


def test_interleaved_conversion_validates_before_launch():
    # from_split / to_split check planes before passing raw pointers
    import torch

    from paper_1401_6235_b200 import interleaved as IL
    from paper_1401_6235_b200 import kernels as K

    v = torch.zeros(8, dtype=torch.float64)
    with pytest.raises(ValueError, match="CUDA tensors"):
        IL.from_split(K.TwofoldArray(v, v))
    with pytest.raises(ValueError, match="CUDA tensors"):
        IL.to_split(torch.zeros((8, 2), dtype=torch.float64))


def test_batch_validation_before_any_launch():
    # kernels.batch / host_batch validate every call (the reference's _check
    # messages) and the batch as a whole before the library is touched
    from paper_1401_6235_b200 import kernels as K

    n = 16
    x = K.TwofoldArray(np.ones(n), np.zeros(n))
    x32 = K.TwofoldArray(np.ones(n, np.float32), np.zeros(n, np.float32))
    o = K.empty_twofold(n, np.float64, device="cpu")
    o32 = K.empty_twofold(n, np.float32, device="cpu")
    K.batch([])
    K.host_batch([])
    with pytest.raises(ValueError, match="mix"):
        K.batch([("vtadd2", x, x, o), ("vtadd2", x32, x32, o32)])
    with pytest.raises(ValueError, match="vtmul2: .*alias"):
        K.host_batch([("vtmul2", x, x, x)])
    with pytest.raises(ValueError, match="lengths differ"):
        K.batch([("vtadd2", x, K.TwofoldArray(np.ones(n + 1), np.zeros(n + 1)), o)])
    with pytest.raises(KeyError):
        K.batch([("vtnope", x, x, o)])
