"""Live cross-check of the oracle against the reference package itself.

Runs only where /root/reference exists (the build container, where the driver
runs the CPU suite); skipped on the GPU box.  Complements the committed goldens
with fresh random inputs drawn over ALL bit patterns (subnormals, infinities,
NaNs, signed zeros included) for every op and both formats, random reduction
geometries, and Horner at random degrees — each compared bit for bit (NaN by
position) with the reference's own numba code (kernels.py:191-247,
demos.py:107-113 style folds on arith.py cores).
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference package not present")


@pytest.fixture(scope="module")
def ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(REF))
    import twofold  # noqa: F401
    from twofold import kernels as RK
    from twofold.fp_core import _div_rem, _sqrt_resid

    return RK, RK._loop11(_div_rem), RK._loop1u(_sqrt_resid)


def _bits_equal(a, b):
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return np.array_equal(a[~na].view(u), b[~nb].view(u))


def _random_bits(rng, n, dtype):
    u = np.uint64 if dtype == np.float64 else np.uint32
    info = np.iinfo(u)
    return rng.integers(0, info.max, n, dtype=u, endpoint=True).view(dtype)


def _mixed(rng, n, dtype):
    # half raw bit patterns (every class of value), half "ordinary" magnitudes
    a = _random_bits(rng, n, dtype)
    b = (rng.uniform(-4, 4, n) * np.exp2(rng.integers(-40, 40, n))).astype(dtype)
    pick = rng.random(n) < 0.5
    return np.where(pick, a, b).astype(dtype)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_every_op_on_random_bit_patterns(oracle, ref, dtype):
    RK, divrem, sqrtres = ref
    rng = np.random.default_rng(2024 if dtype == np.float64 else 2025)
    n = 4000
    names = list(RK.KERNELS) + ["div_rem", "sqrt_resid"]
    for name in names:
        nin = oracle.NUM_INPUTS[name]
        ins = [_mixed(rng, n, dtype) for _ in range(nin)]
        out = RK.empty_twofold(n, dtype)
        with np.errstate(all="ignore"):
            if name == "div_rem":
                divrem(ins[0], ins[1], out.value, out.error)
            elif name == "sqrt_resid":
                sqrtres(ins[0], out.value, out.error)
            else:
                spec = RK.KERNELS[name]
                spec.loop(*ins, out.value, out.error)
            w0, w1 = oracle.elementwise(name, *ins, nthreads=2)
        assert _bits_equal(w0, out.value), name
        assert _bits_equal(w1, out.error), name


def test_reductions_random_geometries(oracle):
    # the canonical fold/tree restated independently in numba on the reference
    # cores (tests/golden/make_golden.py) vs the oracle, at random geometries
    golden = Path(__file__).resolve().parent / "golden"
    sys.path.insert(0, str(golden))
    import make_golden as mg

    rng = np.random.default_rng(77)
    for trial in range(12):
        V = int(rng.choice([1, 2, 4]))
        W = int(rng.choice([1, 3, 8, 32]))
        K = int(rng.choice([1, 2, 5]))
        L = V * W * K
        n = int(rng.integers(0, 9 * L + 3))
        dtype = np.float64 if trial % 2 == 0 else np.float32
        x = _mixed(rng, n, dtype)
        y = _mixed(rng, n, dtype)
        finite = np.isfinite(x) & np.isfinite(y)
        x, y = np.where(finite, x, 1).astype(dtype), np.where(finite, y, 1).astype(dtype)
        for rop, code in (("sum", 0), ("sum2", 1), ("dot", 2)):
            with np.errstate(all="ignore"):
                z0, z1, _, _ = mg._ref_reduce(code, x, y, V, W, K)
                w = oracle.reduce(rop, x, None if rop == "sum" else y, geometry=(V, W, K))
            assert _bits_equal(np.array([w[0], w[1]]), np.array([z0, z1], dtype)), (rop, V, W, K, n)


def test_horner_random_degrees(oracle):
    golden = Path(__file__).resolve().parent / "golden"
    sys.path.insert(0, str(golden))
    import make_golden as mg

    rng = np.random.default_rng(5)
    for deg in (0, 1, 3, 7, 20, 33):
        for dtype in (np.float64, np.float32):
            c = rng.uniform(-3, 3, deg + 1).astype(dtype)
            x = rng.uniform(-2, 2, 513).astype(dtype)
            with np.errstate(all="ignore"):
                o0, o1 = mg._ref_horner(c, x)
                w0, w1 = oracle.horner(c.astype(np.float64), x, nthreads=2)
            assert _bits_equal(w0, o0) and _bits_equal(w1, o1), (deg, dtype)
