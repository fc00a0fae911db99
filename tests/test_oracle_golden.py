"""Pin the CPU oracle against the reference's own outputs (CPU-only tests).

The fixtures under tests/golden/ were produced by the reference package's numba
code (tests/golden/make_golden.py).  The oracle must reproduce them bit for bit
(NaN positions compared by isnan, as test_kernels.py:148-155 does) before any
GPU result is compared against it.
"""

import hashlib
import json
import math
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN

ELEM = np.load(GOLDEN / "elementwise.npz")
RED = np.load(GOLDEN / "reductions.npz")
RED_CASES = json.loads((GOLDEN / "reductions.json").read_text())
HORNER = np.load(GOLDEN / "horner.npz")
KAT = json.loads((GOLDEN / "accumulate_kat.json").read_text())

NAMES = sorted({k.split("/")[0] for k in ELEM.files})


def bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return np.array_equal(a[~na].view(u), b[~nb].view(u))


def test_golden_covers_registry_and_raw_loops():
    assert len(NAMES) == 24  # 22 registry kernels + div_rem + sqrt_resid


@pytest.mark.parametrize("fmt", ["f64", "f32"])
@pytest.mark.parametrize("name", NAMES)
def test_oracle_elementwise_matches_reference(oracle, name, fmt):
    ins = []
    k = 0
    while "%s/%s/in%d" % (name, fmt, k) in ELEM.files:
        ins.append(ELEM["%s/%s/in%d" % (name, fmt, k)])
        k += 1
    with np.errstate(all="ignore"):
        r0, r1 = oracle.elementwise(name, *ins, nthreads=2)
    assert bits_equal(r0, ELEM["%s/%s/out0" % (name, fmt)]), name
    assert bits_equal(r1, ELEM["%s/%s/out1" % (name, fmt)]), name


def _regen(case):
    dtype = np.float64 if case["fmt"] == "f64" else np.float32
    n = case["n"]
    if case["stored"]:
        return RED[case["key"] + "/x"], RED[case["key"] + "/y"]
    rng = np.random.default_rng(case["seed"])
    if case["kind"] == "uniform":
        x = rng.uniform(-1, 1, n)
        y = rng.uniform(-1, 1, n)
    else:
        x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))
        y = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))
    x, y = x.astype(dtype), y.astype(dtype)
    if case["rop"] == "sum2":
        y = (x * dtype(2.0**-30) * y).astype(dtype)
    h = hashlib.sha256()
    h.update(x.tobytes())
    h.update(y.tobytes())
    assert h.hexdigest() == case["sha"], "regenerated inputs differ from the golden run"
    return x, y


@pytest.mark.parametrize("case", RED_CASES, ids=[c["key"] for c in RED_CASES])
def test_oracle_reduction_matches_reference_order(oracle, case):
    x, y = _regen(case)
    b = None if case["rop"] == "sum" else y
    z0, z1, tiles = oracle.reduce(case["rop"], x, b, geometry=tuple(case["geom"]),
                                  nthreads=2, tiles=True)
    want = RED[case["key"] + "/z"]
    assert bits_equal(np.array([z0, z1]), want)
    assert bits_equal(tiles, RED[case["key"] + "/tiles"])


def test_oracle_reduction_bound_holds(oracle):
    # |(z0+z1) - exact| <= 4u·Σ|terms| on the golden cases with n > 0
    for case in RED_CASES[::7]:
        if case["n"] == 0:
            continue
        x, y = _regen(case)
        z = RED[case["key"] + "/z"]
        b = None if case["rop"] == "sum" else y
        ok, err, s, t = oracle.bound_ok(z[0], z[1], case["rop"], x, b,
                                        dtype=x.dtype)
        assert ok, (case["key"], float(err), float(t))


@pytest.mark.parametrize("fmt", ["f64", "f32"])
@pytest.mark.parametrize("deg", [20, 5, 1, 0])
def test_oracle_horner_matches_reference(oracle, fmt, deg):
    x = HORNER["%s/deg%d/x" % (fmt, deg)]
    c = HORNER["%s/deg%d/c" % (fmt, deg)]
    o0, o1 = oracle.horner(c, x, nthreads=2)
    assert bits_equal(o0, HORNER["%s/deg%d/out0" % (fmt, deg)])
    assert bits_equal(o1, HORNER["%s/deg%d/out1" % (fmt, deg)])


@pytest.mark.parametrize("kat", KAT, ids=["%s-%dh" % (k["fmt"], k["hours"]) for k in KAT])
def test_sequential_geometry_reproduces_accumulate(oracle, kat):
    # one tile, one lane: the canonical order degenerates to _accumulate's
    # serial fold (demos.py:107-113)
    dtype = np.float64 if kat["fmt"] == "f64" else np.float32
    n = kat["steps"]
    x0 = np.full(n, kat["t0"], dtype)
    x1 = np.full(n, kat["t1"], dtype)
    z0, z1 = oracle.reduce("sum2", x0, x1, geometry=(1, 1, n))
    assert (float(z0), float(z1)) == (kat["s0"], kat["s1"])


def test_sum100h_transcript_values(oracle):
    # demos.sum100h renders the counter in hours: 100[3.33695e-09] (f64) and
    # 96.3958[3.54008] (f32), goldens sum100h_f64_100h.txt / _f32_100h.txt
    kat = {(k["fmt"], k["hours"]): k for k in KAT}
    k = kat[("f64", 100)]
    n = k["steps"]
    z0, z1 = oracle.reduce("sum2", np.full(n, 0.1), np.zeros(n), geometry=(1, 1, n))
    assert "%.6g[%.6g]" % (z0 / 3600.0, z1 / 3600.0) == "100[3.33695e-09]"
    t0, t1 = np.float32(k["t0"]), np.float32(kat[("f32", 100)]["t1"])
    z0, z1 = oracle.reduce("sum2", np.full(n, np.float32(0.1)), np.full(n, t1, np.float32),
                           geometry=(1, 1, n))
    shown = (np.float32(z0) / np.float32(3600), np.float32(z1) / np.float32(3600))
    assert "%.6g[%.6g]" % (float(shown[0]), float(shown[1])) == "96.3958[3.54008]"
    del t0


# ---- known-answer tests transcribed from the reference's own test files ----

EPS = 2.0**-53


def _one(oracle, name, *args, dtype=np.float64):
    planes = [np.array([a], dtype=dtype) for a in args]
    with np.errstate(all="ignore"):
        r0, r1 = oracle.elementwise(name, *planes, nthreads=1)
    return float(r0[0]), float(r1[0])


def test_kat_acceptance_worked_examples(oracle):
    # test_acceptance.py:333-352
    assert _one(oracle, "vtadd2", 1.0, -EPS, EPS, -(EPS * EPS)) == (1.0, 0.0)
    assert _one(oracle, "vtdiv2", 1.0, 0.0, 1.0 - EPS, EPS) == (1.0 + 2 * EPS, -2 * EPS)
    z = _one(oracle, "vtsqrt1", 1.0, 1.0)
    assert z == (1.0, 0.41421356237309503)
    assert _one(oracle, "vtdiv1", 1.0, 1.0, 1.0) == (1.0, 1.0)


def test_kat_arith_examples(oracle):
    # test_arith.py:89-95, 121-126, 173-201
    a = 1.0 + 2.0**-27
    assert _one(oracle, "vtmul2", a, 0.0, a, 0.0) == (1.0 + 2.0**-26, 2.0**-54)
    assert _one(oracle, "vtmul1", 1.0, EPS, 3.0) == (3.0, 3 * EPS)
    assert _one(oracle, "vtdiv", 6.0, 3.0) == (2.0, 0.0)
    v, e = _one(oracle, "vtdiv", 1.0, 0.0)
    assert v == math.inf and math.isnan(e)
    assert _one(oracle, "vtsqrt", 4.0) == (2.0, 0.0)
    v, e = _one(oracle, "vtsqrt", -1.0)
    assert math.isnan(v) and math.isnan(e)
    v, e = _one(oracle, "vtsqrt", 0.0)
    assert v == 0.0 and math.isnan(e)
    v, e = _one(oracle, "vtsqrt", -0.0)
    assert v == 0.0 and math.copysign(1, v) < 0 and math.isnan(e)
    v, e = _one(oracle, "vtsqrt", math.inf)
    assert v == math.inf and math.isnan(e)


def test_kat_fma_probe(oracle):
    # _fused_or_die probes (fp_core.py:104-119) through TwoProd's residual
    a = 1.0 + 2.0**-27
    p, e = _one(oracle, "vtmul", a, a)
    assert Fraction(p) + Fraction(e) == Fraction(a) * Fraction(a)
    a32 = np.float32(1.0 + 2.0**-12)
    p, e = _one(oracle, "vtmul", a32, a32, dtype=np.float32)
    assert Fraction(p) + Fraction(e) == Fraction(float(a32)) ** 2


def test_kernel_specials(oracle):
    # test_kernels.py:143-155
    with np.errstate(all="ignore"):
        v, e = oracle.elementwise("vtdiv", np.array([1.0, 0.0, -1.0]), np.array([0.0, 0.0, np.inf]))
    assert v[0] == np.inf and np.isnan(e[0])
    assert np.isnan(v[1]) and np.isnan(e[1])
    assert v[2] == 0.0 and np.signbit(v[2])


def test_exact_accumulator_against_fractions(oracle):
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, 500) * np.exp2(rng.integers(-200, 200, 500))
    y = rng.uniform(-1, 1, 500) * np.exp2(rng.integers(-200, 200, 500))
    s, t = oracle.exact("sum", x)
    assert s == sum(Fraction(float(v)) for v in x)
    assert t == sum(abs(Fraction(float(v))) for v in x)
    s, t = oracle.exact("dot", x, y)
    assert s == sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y))
    sub = np.array([5e-324, -5e-324, 2.5e-308, 1e308, -1e308], np.float64)
    s, _ = oracle.exact("dot", sub, sub)
    assert s == sum(Fraction(float(a)) ** 2 for a in sub)
    x32 = (rng.uniform(-1, 1, 500) * np.exp2(rng.integers(-140, 120, 500))).astype(np.float32)
    s, _ = oracle.exact("sum2", x32, x32)
    assert s == 2 * sum(Fraction(float(v)) for v in x32)
