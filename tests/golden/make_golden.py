"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every output in the fixtures is produced by the reference's own numba code:

* elementwise: ``twofold.kernels.KERNELS[name].func`` (kernels.py:191-247), plus
  the raw exact-transform loops ``_loop11(_div_rem)`` / ``_loop1u(_sqrt_resid)``
  exactly as test_acceptance.py:42-43 drives them;
* reductions: the canonical order of DESIGN.md written here in numba on top of
  the reference cores ``_tadd1``/``_tadd``/``_two_prod`` (arith.py:61-71,
  fp_core.py:170-173) — an implementation independent of oracle/twofold_oracle.c;
* Horner: per point ``_tadd1(_tmul1(r, x), c_k)`` with the reference cores;
* the sequential fold KAT: ``twofold.demos._accumulate`` (demos.py:107-113).

Inputs are stored with the outputs (small cases) or as (seed, n, sha256) so a
test can regenerate and verify them (large seeded cases).  The GPU box never
runs this script; it only reads the committed .npz files.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import twofold as tf  # noqa: E402
from numba import njit  # noqa: E402
from twofold import bench  # noqa: E402
from twofold.arith import _tadd, _tadd1, _tmul1  # noqa: E402
from twofold.demos import _accumulate, twofold_from_decimal  # noqa: E402
from twofold.fp_core import _div_rem, _sqrt_resid, _two_prod  # noqa: E402
from twofold.kernels import KERNELS, TwofoldArray, _loop11, _loop1u, empty_twofold  # noqa: E402

OUT = Path(__file__).resolve().parent
FMTS = {"f64": np.float64, "f32": np.float32}

_div_rem_loop = _loop11(_div_rem)
_sqrt_resid_loop = _loop1u(_sqrt_resid)


# --------------------------------------------------------------------------
# elementwise


def _planes(rng, n, dtype, positive=False, coupled=False):
    # same shape of distribution as test_kernels.py:27-37
    v = rng.uniform(1, 2, n) * np.exp2(rng.integers(-3, 4, n))
    if not positive:
        v = v * rng.choice([-1.0, 1.0], n)
    v = v.astype(dtype)
    if coupled:
        scale = 2.0**-25 if dtype == np.float32 else 2.0**-54
    else:
        scale = 2.0**-24 if dtype == np.float32 else 2.0**-52
    e = (v * scale * rng.uniform(-1, 1, n).astype(dtype)).astype(dtype)
    return v, e


def _wide(rng, n, dtype, max_exp):
    # test_acceptance.py:185-187
    mag = rng.uniform(1, 2, n) * np.exp2(rng.integers(-max_exp, max_exp + 1, n))
    return (mag * rng.choice([-1.0, 1.0], n)).astype(dtype)


def _corners(dtype):
    # test_acceptance.py:286-295
    if dtype == np.float64:
        c = [0.0, -0.0, 1.0, -1.5, math.inf, -math.inf, math.nan,
             5e-324, -5e-324, 6.5e-310, 1.7976931348623157e308]
    else:
        c = [float(np.float32(s)) for s in
             ["0", "-0", "1", "-1.5", "inf", "-inf", "nan",
              "1.401298464324817e-45", "-1.401298464324817e-45",
              "9.2e-41", "3.4028234663852886e38"]]
    return np.array(c, dtype=dtype)


def _arity(name):
    if name == "div_rem":
        return "11"
    if name == "sqrt_resid":
        return "u1"
    return KERNELS[name].arity


def _nin(ar):
    return {"22": 4, "21": 3, "11": 2, "u2": 2, "u1": 1}[ar]


def _inputs(name, fmt, rng):
    dtype = FMTS[fmt]
    ar = _arity(name)
    k = _nin(ar)
    coupled = name.startswith("vp")
    positive = name in ("vtsqrt1", "vtsqrt", "sqrt_resid")
    cols = [[] for _ in range(k)]

    def add(*planes):
        for c, p in zip(cols, planes):
            c.append(np.asarray(p, dtype=dtype))

    # (a) test_kernels-style planes, n=256
    n = 256
    if ar == "22":
        x = _planes(rng, n, dtype, coupled=coupled)
        y = _planes(rng, n, dtype, coupled=coupled)
        add(x[0], x[1], y[0], y[1])
    elif ar == "21":
        x = _planes(rng, n, dtype, coupled=coupled)
        add(x[0], x[1], _planes(rng, n, dtype)[0])
    elif ar == "11":
        add(_planes(rng, n, dtype)[0], _planes(rng, n, dtype)[0])
    elif ar == "u2":
        add(*_planes(rng, n, dtype, positive=True, coupled=coupled))
    else:
        add(_planes(rng, n, dtype, positive=True)[0])
    # (b) the reference bench's inputs (bench.py:144-162), n=128
    if name in KERNELS:
        add(*bench._inputs(name, fmt, 128))
    # (c) wide exponents (crit 4/7 style), n=128, tails 2^-60..2^2 below heads
    n = 128
    me = 150 if fmt == "f64" else 15
    heads = [_wide(rng, n, dtype, me) for _ in range(2)]
    if positive:
        heads = [np.abs(h) for h in heads]
    with np.errstate(all="ignore"):
        tails = [(h * np.exp2(-rng.integers(-2, 61, n)) * rng.choice([-1.0, 1.0], n)).astype(dtype)
                 for h in heads]
    if ar == "22":
        add(heads[0], tails[0], heads[1], tails[1])
    elif ar == "21":
        add(heads[0], tails[0], heads[1])
    elif ar == "11":
        add(heads[0], heads[1])
    elif ar == "u2":
        add(heads[0], tails[0])
    else:
        add(heads[0])
    # (d) IEEE corners, full cross product (121 cases), zero error planes,
    # then the same heads with unit-scale error planes
    c = _corners(dtype)
    a = np.repeat(c, len(c))
    b = np.tile(c, len(c))
    z = np.zeros_like(a)
    one = np.ones_like(a)
    if ar == "22":
        add(a, z, b, z)
        add(a, one, b, -one)
    elif ar == "21":
        add(a, z, b)
        add(a, b, one)
    elif ar == "11":
        add(a, b)
    elif ar == "u2":
        add(a, z)
        add(a, b)
    else:
        add(c)
    return [np.concatenate(col) for col in cols]


def _run_reference(name, ins, dtype):
    n = ins[0].shape[0]
    if name == "div_rem":
        out = empty_twofold(n, dtype)
        _div_rem_loop(ins[0], ins[1], out.value, out.error)
        return out.value, out.error
    if name == "sqrt_resid":
        out = empty_twofold(n, dtype)
        _sqrt_resid_loop(ins[0], out.value, out.error)
        return out.value, out.error
    spec = KERNELS[name]
    out = empty_twofold(n, dtype, spec.out_kind)
    with np.errstate(all="ignore"):
        if spec.arity == "22":
            spec.func(TwofoldArray(ins[0], ins[1]), TwofoldArray(ins[2], ins[3]), out)
        elif spec.arity == "21":
            spec.func(TwofoldArray(ins[0], ins[1]), ins[2], out)
        elif spec.arity == "11":
            spec.func(ins[0], ins[1], out)
        elif spec.arity == "u2":
            spec.func(TwofoldArray(ins[0], ins[1]), out)
        else:
            spec.func(ins[0], out)
    return out.value, out.error


def make_elementwise():
    data = {}
    names = list(KERNELS) + ["div_rem", "sqrt_resid"]
    for fmt, dtype in FMTS.items():
        for j, name in enumerate(names):
            rng = np.random.default_rng(1000 + 31 * j + (0 if fmt == "f64" else 7))
            ins = _inputs(name, fmt, rng)
            r0, r1 = _run_reference(name, ins, dtype)
            for k, p in enumerate(ins):
                data["%s/%s/in%d" % (name, fmt, k)] = p
            data["%s/%s/out0" % (name, fmt)] = r0
            data["%s/%s/out1" % (name, fmt)] = r1
    np.savez_compressed(OUT / "elementwise.npz", **data)
    print("elementwise.npz:", len(data), "arrays")


# --------------------------------------------------------------------------
# reductions in the canonical order, on the reference cores


@njit(cache=False)
def _tree(a0, a1, m):
    stride = 1
    while stride < m:
        i = 0
        while i + stride < m:
            a0[i], a1[i] = _tadd(a0[i], a1[i], a0[i + stride], a1[i + stride])
            i += 2 * stride
        stride *= 2
    return a0[0], a1[0]


@njit(cache=False)
def _ref_reduce(rop, a, b, V, W, K):
    n = a.shape[0]
    L = V * W * K
    T = (n + L - 1) // L
    t0 = np.zeros(max(T, 1), a.dtype)
    t1 = np.zeros(max(T, 1), a.dtype)
    l0 = np.zeros(W, a.dtype)
    l1 = np.zeros(W, a.dtype)
    zero = np.zeros(1, a.dtype)[0]
    for t in range(T):
        m = 0
        for w in range(W):
            have = False
            s0 = zero
            s1 = zero
            for k in range(K):
                for v in range(V):
                    i = t * L + V * (w + W * k) + v
                    if i >= n:
                        continue
                    if rop == 0:
                        if not have:
                            s0 = a[i]
                            s1 = zero
                            have = True
                        else:
                            s0, s1 = _tadd1(s0, s1, a[i])
                    else:
                        if rop == 1:
                            p0 = a[i]
                            p1 = b[i]
                        else:
                            p0, p1 = _two_prod(a[i], b[i])
                        if not have:
                            s0 = p0
                            s1 = p1
                            have = True
                        else:
                            s0, s1 = _tadd(s0, s1, p0, p1)
            if not have:
                break
            l0[m] = s0
            l1[m] = s1
            m += 1
        t0[t], t1[t] = _tree(l0, l1, m)
    if T == 0:
        return zero, zero, t0[:0], t1[:0]
    z0, z1 = _tree(t0.copy(), t1.copy(), T)
    return z0, z1, t0[:T], t1[:T]


def _seeded(kind, seed, n, dtype):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        x = rng.uniform(-1, 1, n)
        y = rng.uniform(-1, 1, n)
    else:  # wide dynamic range with cancellation
        x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))
        y = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))
    return x.astype(dtype), y.astype(dtype)


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def make_reductions():
    cases = []
    small_geoms = [(2, 8, 4), (4, 8, 2), (1, 1, 1), (2, 4, 3)]
    prod = {"f64": (2, 256, 128), "f32": (4, 256, 128)}
    data = {}
    idx = 0
    for fmt, dtype in FMTS.items():
        for rop_name, rop in (("sum", 0), ("sum2", 1), ("dot", 2)):
            for geom in small_geoms + [prod[fmt]]:
                L = geom[0] * geom[1] * geom[2]
                sizes = sorted({0, 1, 2, 3, L - 1, L, L + 1, 2 * L + 5, 7 * L + 3, 16 * L})
                if geom == prod[fmt]:
                    sizes = [0, 1, 5, 1000, L - 3, L, L + 1, 3 * L + 12345, (1 << 24) + 17]
                for n in sizes:
                    kind = "wide" if (idx % 2) else "uniform"
                    seed = 5000 + idx
                    x, y = _seeded(kind, seed, n, dtype)
                    if rop_name == "sum2":
                        y = (x * dtype(2.0**-30) * y).astype(dtype)
                    z0, z1, t0, t1 = _ref_reduce(rop, x, y, *geom)
                    store = n <= 4096
                    key = "r%04d" % idx
                    meta = dict(key=key, fmt=fmt, rop=rop_name, geom=list(geom), n=int(n),
                                kind=kind, seed=seed, sha=_sha(x, y), stored=store)
                    if store:
                        data[key + "/x"] = x
                        data[key + "/y"] = y
                    data[key + "/z"] = np.array([z0, z1], dtype)
                    data[key + "/tiles"] = np.stack([t0, t1], 1).astype(dtype) if n else np.zeros((0, 2), dtype)
                    cases.append(meta)
                    idx += 1
    np.savez_compressed(OUT / "reductions.npz", **data)
    (OUT / "reductions.json").write_text(json.dumps(cases, indent=1))
    print("reductions:", len(cases), "cases")


# --------------------------------------------------------------------------
# Horner and the sequential-fold KAT


@njit(cache=False)
def _ref_horner(c, x):
    n = x.shape[0]
    o0 = np.empty_like(x)
    o1 = np.empty_like(x)
    d = c.shape[0] - 1
    for i in range(n):
        r0 = c[d]
        r1 = c[d] - c[d]
        for k in range(d - 1, -1, -1):
            r0, r1 = _tmul1(r0, r1, x[i])
            r0, r1 = _tadd1(r0, r1, c[k])
        o0[i] = r0
        o1[i] = r1
    return o0, o1


def binom_coeffs(deg=20):
    return [(-1) ** (deg - k) * math.comb(deg, k) for k in range(deg + 1)]


def make_horner():
    data = {}
    for fmt, dtype in FMTS.items():
        rng = np.random.default_rng(77 if fmt == "f64" else 78)
        x = np.concatenate([rng.uniform(0.9, 1.1, 1021),
                            [1.0, 0.0, 2.0, -1.0, 0.5, 1.0 + 2.0**-20]]).astype(dtype)
        for deg in (20, 5, 0, 1):
            c = np.array(binom_coeffs(deg), dtype=dtype)
            o0, o1 = _ref_horner(c, x)
            data["%s/deg%d/x" % (fmt, deg)] = x
            data["%s/deg%d/c" % (fmt, deg)] = c.astype(np.float64)
            data["%s/deg%d/out0" % (fmt, deg)] = o0
            data["%s/deg%d/out1" % (fmt, deg)] = o1
    np.savez_compressed(OUT / "horner.npz", **data)
    print("horner.npz written")


def make_accumulate_kat():
    # demos.py:116-140: hours*36000 steps of the twofold image of 0.1
    kat = []
    for fmt in ("f64", "f32"):
        for hours in (1, 100):
            t = twofold_from_decimal("0.1", fmt)
            steps = hours * 36000
            s0, s1 = _accumulate(t.value, t.error, steps)
            kat.append(dict(fmt=fmt, hours=hours, steps=steps,
                            t0=float(t.value), t1=float(t.error),
                            s0=float(s0), s1=float(s1)))
    (OUT / "accumulate_kat.json").write_text(json.dumps(kat, indent=1))
    print("accumulate KAT:", kat)


if __name__ == "__main__" and len(sys.argv) == 1:
    make_elementwise()
    make_reductions()
    make_horner()
    make_accumulate_kat()


# --------------------------------------------------------------------------
# fused demo chains (demos.py:153-238) through the reference's scalar API


def _ref_quadratic(a, b, c, fmt):
    # demos.py:219-229, the same calls
    four = twofold_from_decimal("4", fmt)
    two = twofold_from_decimal("2", fmt)
    disc = tf.tsub(tf.tmul(b, b), tf.tmul(tf.tmul(four, a), c))
    d = tf.tsqrt(disc)
    neg_b = tf.tneg(b)
    two_a = tf.tmul(two, a)
    x0 = tf.tdiv(tf.tsub(neg_b, d), two_a)
    x1 = tf.tdiv(tf.tadd(neg_b, d), two_a)
    return d, x0, x1


def _ref_gauss3(a, f):
    # demos.py:177-192, the same loops
    a = [row[:] for row in a]
    f = f[:]
    for k in range(3):
        for i in range(k + 1, 3):
            m = tf.tdiv(a[i][k], a[k][k])
            for j in range(k, 3):
                a[i][j] = tf.tsub(a[i][j], tf.tmul(m, a[k][j]))
            f[i] = tf.tsub(f[i], tf.tmul(m, f[k]))
    x = [None, None, None]
    for i in (2, 1, 0):
        s = f[i]
        for j in range(i + 1, 3):
            s = tf.tsub(s, tf.tmul(a[i][j], x[j]))
        x[i] = tf.tdiv(s, a[i][i])
    return x


def make_fused():
    from twofold.demos import _CASES, _parse_c, gauss_solve, quadratic_roots

    data, meta = {}, {}
    for fmt, dtype in FMTS.items():
        T = dtype
        rng = np.random.default_rng(900 if fmt == "f64" else 901)
        n = 512
        tw = lambda v, e: tf.Twofold(T(v), T(e))  # noqa: E731
        # axpy / submul on random twofolds
        planes = [_planes(rng, n, dtype) for _ in range(3)]
        flat = [p for pair in planes for p in pair]
        ax0, ax1, sm0, sm1 = (np.empty(n, dtype) for _ in range(4))
        for i in range(n):
            a, x, y = (tw(planes[k][0][i], planes[k][1][i]) for k in range(3))
            z = tf.tadd(tf.tmul(a, x), y)
            ax0[i], ax1[i] = z
            z = tf.tsub(a, tf.tmul(x, y))
            sm0[i], sm1[i] = z
        for k, p in enumerate(flat):
            data["axpy/%s/in%d" % (fmt, k)] = p
        data["axpy/%s/out" % fmt] = np.stack([ax0, ax1])
        data["submul/%s/out" % fmt] = np.stack([sm0, sm1])
        # quadratic: the demo's three cases, then random coefficients
        cases = ["1e-8", "1+1e-8", "1-1e-8"]
        A = [(T(1), T(0))] * len(cases)
        B = [(T(2), T(0))] * len(cases)
        C = [tuple(twofold_from_decimal(repr(_parse_c(c)), fmt)) for c in cases]
        tokens = []
        for c in cases:
            rep = quadratic_roots(fmt, c).render()
            tokens.append({ln.strip().split(": ")[0]: ln.strip().split(": ")[1]
                           for ln in rep.splitlines() if ": " in ln and not ln.startswith("test")})
        m = 509
        a0 = rng.uniform(0.5, 2, m) * rng.choice([-1.0, 1.0], m)
        b0 = rng.uniform(-4, 4, m)
        c0 = rng.uniform(-1, 1, m)
        A += [(T(v), T(v * 2.0**-30)) for v in a0]
        B += [(T(v), T(-v * 2.0**-31)) for v in b0]
        C += [(T(v), T(v * 2.0**-29)) for v in c0]
        qin = [np.array([p[j] for p in P], dtype) for P in (A, B, C) for j in (0, 1)]
        qout = [np.empty(len(A), dtype) for _ in range(6)]
        for i in range(len(A)):
            d, x0, x1 = _ref_quadratic(tf.Twofold(*A[i]), tf.Twofold(*B[i]), tf.Twofold(*C[i]), fmt)
            for k, z in enumerate((d, x0, x1)):
                qout[2 * k][i], qout[2 * k + 1][i] = z
        for k in range(6):
            data["quad/%s/in%d" % (fmt, k)] = qin[k]
            data["quad/%s/out%d" % (fmt, k)] = qout[k]
        meta["quad/%s" % fmt] = {"cases": cases, "tokens": tokens}
        # gauss3: the demo's two systems, then random diagonally dominant ones
        systems = []
        for case in ("well3", "ill3"):
            lam_t, f_t, _ = _CASES[case]
            lam = twofold_from_decimal(lam_t, fmt)
            one = twofold_from_decimal("1", fmt)
            zero = twofold_from_decimal("0", fmt)
            a = [[lam, one, zero], [zero, lam, one], [zero, zero, lam]]
            f = [twofold_from_decimal(t, fmt) for t in f_t]
            systems.append((a, f))
        gtok = {}
        for case in ("well3", "ill3"):
            sol = gauss_solve(fmt, case).render().splitlines()[-1].split()
            gtok[case] = sol
        for _ in range(254):
            M = rng.uniform(-1, 1, (3, 3)) + 4 * np.eye(3)
            fv = rng.uniform(-5, 5, 3)
            a = [[tw(M[r, c], M[r, c] * 2.0**-40) for c in range(3)] for r in range(3)]
            f = [tw(fv[r], 0.0) for r in range(3)]
            systems.append((a, f))
        ns = len(systems)
        Av = np.empty((3, 3, ns), dtype)
        Ae = np.empty((3, 3, ns), dtype)
        Fv = np.empty((3, ns), dtype)
        Fe = np.empty((3, ns), dtype)
        Xv = np.empty((3, ns), dtype)
        Xe = np.empty((3, ns), dtype)
        for s_, (a, f) in enumerate(systems):
            for r in range(3):
                for c in range(3):
                    Av[r, c, s_], Ae[r, c, s_] = a[r][c]
                Fv[r, s_], Fe[r, s_] = f[r]
            x = _ref_gauss3(a, f)
            for r in range(3):
                Xv[r, s_], Xe[r, s_] = x[r]
        for k, arr in (("Av", Av), ("Ae", Ae), ("Fv", Fv), ("Fe", Fe), ("Xv", Xv), ("Xe", Xe)):
            data["gauss3/%s/%s" % (fmt, k)] = arr
        meta["gauss3/%s" % fmt] = {"tokens": gtok}
    np.savez_compressed(OUT / "fused.npz", **data)
    (OUT / "fused.json").write_text(json.dumps(meta, indent=1))
    print("fused fixtures written")


if __name__ == "__main__" and ("fused" in sys.argv or len(sys.argv) == 1):
    make_fused()


# --------------------------------------------------------------------------
# config-size hashes: the reference's own outputs on BASELINE-distributed inputs


def _cfg_inputs(config, name, n, seed):
    sys.path.insert(0, str(OUT))
    from config_inputs import cfg_inputs

    return cfg_inputs(config, name, n, seed)


def make_config_hashes():
    cases = []
    plan = [("config1", ["vtadd2", "vtmul2"], 1 << 20),
            ("config2", ["vtadd2", "vtsub2", "vtmul2", "vtdiv2", "vtsqrt1"], 1 << 22),
            ("config3", ["vtadd2", "vtmul2", "vtdiv2"], 1 << 22)]
    for config, names, n in plan:
        for j, name in enumerate(names):
            seed = 7000 + 10 * j + int(config[-1])
            ins = _cfg_inputs(config, name, n, seed)
            dtype = ins[0].dtype
            r0, r1 = _run_reference(name, ins, dtype)
            cases.append(dict(config=config, op=name, n=n, seed=seed, dtype=str(dtype),
                              numpy=np.__version__, sha_in=_sha(*ins),
                              sha_z0=hashlib.sha256(r0.tobytes()).hexdigest(),
                              sha_z1=hashlib.sha256(r1.tobytes()).hexdigest()))
    (OUT / "config_hashes.json").write_text(json.dumps(cases, indent=1))
    print("config hashes:", len(cases))


if __name__ == "__main__" and ("hashes" in sys.argv or len(sys.argv) == 1):
    make_config_hashes()
