"""GPU parity of the reductions and Horner (B200).

Reductions: bit-exact against the reference-generated goldens at the device
geometry and against the oracle at larger sizes; the error bound
|(z0+z1) - exact| <= 4u·Σ|terms| against the exact accumulator; bit-identical
results for every shard count G (shards reduced on the device and combined
with tf_combine, as the multi-GPU path does).
"""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import GOLDEN  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

RED = np.load(GOLDEN / "reductions.npz")
RED_CASES = json.loads((GOLDEN / "reductions.json").read_text())
HORNER = np.load(GOLDEN / "horner.npz")


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV)


def _device_reduce(rop, x, y=None, offset=0):
    from paper_1401_6235_b200 import reduce as R

    def put(a):
        if offset == 0:
            return _t(a)
        buf = torch.empty(a.shape[0] + offset, dtype=_t(a[:1]).dtype, device=DEV)
        buf[offset:].copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return buf[offset:]

    if rop == "sum":
        z = R.vtsum(put(x))
    elif rop == "sum2":
        z = R.vtsum2((put(x), put(y)))
    else:
        z = R.vtdot(put(x), put(y))
    return z


def _geom(dtype):
    from paper_1401_6235_b200 import reduce as R

    return R.geometry(dtype)


def _regen(case):
    dtype = np.float64 if case["fmt"] == "f64" else np.float32
    if case["stored"]:
        return RED[case["key"] + "/x"], RED[case["key"] + "/y"]
    n = case["n"]
    rng = np.random.default_rng(case["seed"])
    if case["kind"] == "uniform":
        x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    else:
        x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))
        y = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))
    x, y = x.astype(dtype), y.astype(dtype)
    if case["rop"] == "sum2":
        y = (x * dtype(2.0**-30) * y).astype(dtype)
    return x, y


DEVICE_CASES = [c for c in RED_CASES if tuple(c["geom"]) in ((2, 256, 128), (4, 256, 128))]


def test_device_geometry_is_the_golden_geometry():
    assert _geom(np.float64) == (2, 256, 128)
    assert _geom(np.float32) == (4, 256, 128)
    assert len(DEVICE_CASES) >= 40


@pytest.mark.parametrize("case", DEVICE_CASES, ids=[c["key"] for c in DEVICE_CASES])
def test_device_reduction_matches_reference_golden(case):
    x, y = _regen(case)
    z = _device_reduce(case["rop"], x, y)
    want = RED[case["key"] + "/z"]
    got = np.array([z.value, z.error], dtype=want.dtype)
    assert np.array_equal(got.view(np.uint64 if want.dtype == np.float64 else np.uint32),
                          want.view(np.uint64 if want.dtype == np.float64 else np.uint32)), (got, want)


@pytest.mark.parametrize("offset", [1, 3])
@pytest.mark.parametrize("rop", ["sum", "sum2", "dot"])
def test_device_reduction_unaligned_planes(oracle, rop, offset):
    rng = np.random.default_rng(offset)
    n = 3 * 65536 + 999
    x = rng.uniform(-1, 1, n)
    y = rng.uniform(-1, 1, n)
    z = _device_reduce(rop, x, y, offset=offset)
    w = oracle.reduce(rop, x, None if rop == "sum" else y, geometry=_geom(np.float64))
    assert (z.value, z.error) == (float(w[0]), float(w[1]))


@pytest.mark.parametrize("fmt", ["f64", "f32"])
@pytest.mark.parametrize("rop", ["sum", "sum2", "dot"])
def test_device_reduction_large_vs_oracle(oracle, rop, fmt):
    dtype = np.float64 if fmt == "f64" else np.float32
    rng = np.random.default_rng(11)
    n = (1 << 24) + 12345
    x = (rng.uniform(-1, 1, n) * np.exp2(rng.integers(-20, 21, n))).astype(dtype)
    y = (rng.uniform(-1, 1, n) * np.exp2(rng.integers(-20, 21, n))).astype(dtype)
    z = _device_reduce(rop, x, y)
    w = oracle.reduce(rop, x, None if rop == "sum" else y, geometry=_geom(dtype))
    assert (z.value, z.error) == (float(w[0]), float(w[1]))


def _ill_dot(n, cond, seed):
    from paper_1401_6235_b200 import _lib

    x = np.empty(n)
    y = np.empty(n)
    assert _lib.lib().tf_gen_dot_host(n, cond, seed, x.ctypes.data, y.ctypes.data) == 0
    return x, y


@pytest.mark.parametrize("cond", [1e8, 1e16, 1e24])
def test_ill_conditioned_dot_and_sum_bound(oracle, cond):
    n = 1 << 21
    x, y = _ill_dot(n, cond, 7)
    z = _device_reduce("dot", x, y)
    w = oracle.reduce("dot", x, y, geometry=_geom(np.float64))
    assert (z.value, z.error) == (float(w[0]), float(w[1]))
    ok, err, s, t = oracle.bound_ok(z.value, z.error, "dot", x, y)
    assert ok, (float(err), float(t))
    achieved = float(2 * t / abs(s)) if s else float("inf")
    assert cond / 2 < achieved < cond * 2  # the generator reaches the requested conditioning
    # the sum form: terms are the exact TwoProd pieces of the products
    p, e = oracle.elementwise("vtmul", x, y)
    terms = np.empty(2 * n)
    terms[0::2] = p
    terms[1::2] = e
    zs = _device_reduce("sum", terms)
    ws = oracle.reduce("sum", terms, geometry=_geom(np.float64))
    assert (zs.value, zs.error) == (float(ws[0]), float(ws[1]))
    ok, err, s2, t2 = oracle.bound_ok(zs.value, zs.error, "sum", terms)
    assert ok and s2 == s


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_shard_count_invariance(G):
    # the multi-GPU data path on one device: each shard reduced by the device
    # kernel, partials combined by tf_combine, must equal the one-shard result
    from paper_1401_6235_b200 import dist as D
    from paper_1401_6235_b200 import reduce as R

    rng = np.random.default_rng(G)
    n = 9 * 65536 + 4321
    x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-40, 41, n))
    X = _t(x)
    whole = R.vtsum(X)
    L = R.tile_elems(np.float64)
    parts = torch.zeros((G, 2), dtype=torch.float64, device=DEV)
    counts = []
    for r in range(G):
        lo, hi = D.shard_tiles(n, G, r, L)
        counts.append(hi - lo)
        if hi > lo:
            R.vtsum(X[lo:hi], out=parts[r])
    z = R.combine(parts, counts)
    assert (z.value, z.error) == (whole.value, whole.error)


def test_empty_and_single():
    from paper_1401_6235_b200 import reduce as R

    z = R.vtsum(torch.empty(0, dtype=torch.float64, device=DEV))
    assert (z.value, z.error) == (0.0, 0.0)
    z = R.vtsum(_t(np.array([-0.0])))
    assert z.value == 0.0 and np.signbit(z.value)  # seeded from (x, +0), not (+0, +0)
    z = R.vtdot(_t(np.array([3.0])), _t(np.array([1.0 / 3.0])))
    assert z.value == 3.0 * (1.0 / 3.0)


@pytest.mark.parametrize("fmt", ["f64", "f32"])
@pytest.mark.parametrize("deg", [20, 5, 1, 0])
def test_horner_matches_reference_golden(fmt, deg):
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R

    x = HORNER["%s/deg%d/x" % (fmt, deg)]
    c = HORNER["%s/deg%d/c" % (fmt, deg)]
    dt = torch.float64 if fmt == "f64" else torch.float32
    out = K.empty_twofold(x.shape[0], dt)
    R.vthorner(c, _t(x), out)
    w0, w1 = HORNER["%s/deg%d/out0" % (fmt, deg)], HORNER["%s/deg%d/out1" % (fmt, deg)]
    u = np.uint64 if fmt == "f64" else np.uint32
    assert np.array_equal(out.value.cpu().numpy().view(u), w0.view(u))
    assert np.array_equal(out.error.cpu().numpy().view(u), w1.view(u))


def test_horner_config5_vs_oracle_and_flag(oracle):
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R

    n = (1 << 22) + 7
    x = np.random.default_rng(5).uniform(0.9, 1.1, n)
    c = R.binomial_coeffs(20)
    out = K.empty_twofold(n, torch.float64)
    R.vthorner(c, _t(x), out)
    w0, w1 = oracle.horner(c, x)
    z0, z1 = out.value.cpu().numpy(), out.error.cpu().numpy()
    assert np.array_equal(z0.view(np.uint64), w0.view(np.uint64))
    assert np.array_equal(z1.view(np.uint64), w1.view(np.uint64))
    nz = z0 != 0
    flag = np.abs(z1[nz]) >= 0.5 * np.abs(z0[nz])
    assert flag.mean() > 0.99  # z1 flags the catastrophic cancellation near x=1


def test_horner_generic_degree_vs_oracle(oracle):
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R

    n = 100_003
    rng = np.random.default_rng(8)
    x = rng.uniform(-2, 2, n)
    c = list(rng.uniform(-1, 1, 37))
    out = K.empty_twofold(n, torch.float64)
    R.vthorner(c, _t(x), out)
    w0, w1 = oracle.horner(c, x)
    assert np.array_equal(out.value.cpu().numpy().view(np.uint64), w0.view(np.uint64))
    assert np.array_equal(out.error.cpu().numpy().view(np.uint64), w1.view(np.uint64))


def _bits_eq_nan(a, b):
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(u), b[~nb].view(u))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("deg", [20, 7])
def test_horner_specials_bit_exact(oracle, dt, deg):
    # Horner through every IEEE corner: zero and -0 operands, infinities, NaN,
    # overflow to inf (and TwoSum intermediates overflowing in the top binade
    # while the sum stays finite), subnormals, and steps whose error is exactly 0
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R

    rng = np.random.default_rng(deg)
    big = np.finfo(dt).max
    tiny = np.finfo(dt).smallest_subnormal
    xs = np.array([0.0, -0.0, 1.0, -1.0, 2.0, 0.5, np.inf, -np.inf, np.nan, big, -big, tiny,
                   -tiny, 1e-30, 3.0, 1.0 + 2**-20], dtype=dt)
    coeff_sets = [
        R.binomial_coeffs(deg),
        [0.0] * (deg + 1),
        [-0.0] * (deg + 1),
        [(-0.0 if k % 2 else 0.0) for k in range(deg + 1)],
        [(1.0 if k % 3 == 0 else -0.0) for k in range(deg + 1)],
        [float(big)] * (deg + 1),
        [float(tiny) * (k + 1) for k in range(deg + 1)],
        [np.inf] + [1.0] * deg,
        [1.0] * deg + [np.nan],
        list(rng.integers(-3, 4, deg + 1).astype(float)),
    ]
    x = np.concatenate([xs, rng.uniform(-3, 3, 4096).astype(dt),
                        rng.integers(-2, 3, 1024).astype(dt)])
    for c in coeff_sets:
        c = [float(v) for v in np.asarray(c, dtype=dt)]
        out = K.empty_twofold(x.shape[0], torch.float64 if dt == np.float64 else torch.float32)
        R.vthorner(c, _t(x), out)
        w0, w1 = oracle.horner(c, x)
        assert _bits_eq_nan(out.value.cpu().numpy(), w0), c[:3]
        assert _bits_eq_nan(out.error.cpu().numpy(), w1), c[:3]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("pin", [False, True])
@pytest.mark.parametrize("rop", ["sum", "sum2", "dot"])
def test_host_plane_reductions_match_device(oracle, rop, pin, dtype):
    # numpy planes go through tf_reduce_host (chunked subtrees + combine): the
    # bits must equal the device-plane reduction and the oracle
    from paper_1401_6235_b200 import reduce as R

    rng = np.random.default_rng(99)
    n = 37 * 65536 + 12345  # several pipeline chunks plus a partial tile
    x = (rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))).astype(dtype)
    y = rng.uniform(-1, 1, n).astype(dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    if pin:
        xp = torch.empty(n, dtype=tdt, pin_memory=True).numpy()
        yp = torch.empty(n, dtype=tdt, pin_memory=True).numpy()
        xp[:] = x
        yp[:] = y
        x, y = xp, yp
    fn = {"sum": lambda a, b: R.vtsum(a), "sum2": lambda a, b: R.vtsum2((a, b)),
          "dot": lambda a, b: R.vtdot(a, b)}[rop]
    zh = fn(x, y)
    zd = fn(_t(x), _t(y))
    w = oracle.reduce(rop, x, None if rop == "sum" else y, geometry=_geom(dtype))
    assert (zh.value, zh.error) == (zd.value, zd.error) == (float(w[0]), float(w[1]))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("pin", [False, True])
def test_host_reduction_batch_matches_single_calls(oracle, pin, dtype):
    # several reductions in one pass over shared host planes (x crosses once):
    # every result equals the single call and the oracle, in call order
    from paper_1401_6235_b200 import reduce as R

    rng = np.random.default_rng(31)
    n = 21 * 131072 + 999
    tdt = torch.float64 if dtype == np.float64 else torch.float32

    def plane(a):
        a = a.astype(dtype)
        if not pin:
            return a
        p = torch.empty(n, dtype=tdt, pin_memory=True).numpy()
        p[:] = a
        return p

    x = plane(rng.uniform(-1, 1, n) * np.exp2(rng.integers(-25, 26, n)))
    y = plane(rng.uniform(-1, 1, n))
    e = plane(x * 2.0**-40 * rng.uniform(-1, 1, n))
    calls = [("vtdot", x, y), ("vtsum", x), ("vtsum2", (x, e)), ("vtdot", y, y), ("vtsum", y)]
    got = R.host_batch(calls)
    g = _geom(dtype)
    want = [oracle.reduce("dot", x, y, geometry=g), oracle.reduce("sum", x, geometry=g),
            oracle.reduce("sum2", x, e, geometry=g), oracle.reduce("dot", y, y, geometry=g),
            oracle.reduce("sum", y, geometry=g)]
    single = [R.vtdot(x, y), R.vtsum(x), R.vtsum2((x, e)), R.vtdot(y, y), R.vtsum(y)]
    for z, w, s1 in zip(got, want, single):
        assert (z.value, z.error) == (float(w[0]), float(w[1])) == (s1.value, s1.error)
    assert R.host_batch([]) == []
    with pytest.raises(ValueError, match="plane lengths differ"):
        R.host_batch([("vtsum", x), ("vtsum", y[:-1])])
    with pytest.raises(ValueError, match="unknown reduction"):
        R.host_batch([("vtmax", x)])
    z0 = R.host_batch([("vtsum", x[:0]), ("vtdot", x[:0], y[:0])])
    assert all(np.copysign(1, v.value) == 1 and v.value == 0 and v.error == 0 for v in z0)


def test_host_plane_reduction_f32_then_f64_fresh_process():
    # the host-reduction staging is sized by the first call; an f64 call after an
    # f32 one (same chunk bytes, twice the tile-partial bytes) must regrow it
    import subprocess
    import sys

    code = (
        "import numpy as np, torch\n"
        "from paper_1401_6235_b200 import reduce as R\n"
        "rng = np.random.default_rng(5)\n"
        "n = 9 * 131072 + 3\n"
        "x32 = rng.uniform(-1, 1, n).astype(np.float32)\n"
        "x64 = rng.uniform(-1, 1, n)\n"
        "for x in (x32, x64, x32):\n"
        "    zh = R.vtsum(x); zd = R.vtsum(torch.as_tensor(x, device='cuda'))\n"
        "    assert (zh.value, zh.error) == (zd.value, zd.error), (zh, zd)\n"
        "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=str(GOLDEN.parents[1]))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_horner_host_planes_match_device(oracle):
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R

    n = 3 * (1 << 22) + 5
    x = np.random.default_rng(12).uniform(0.9, 1.1, n)
    c = R.binomial_coeffs(20)
    out = K.empty_twofold(n, np.float64, device="cpu")
    R.vthorner(c, x, out)
    w0, w1 = oracle.horner(c, x)
    assert np.array_equal(out.value.view(np.uint64), w0.view(np.uint64))
    assert np.array_equal(out.error.view(np.uint64), w1.view(np.uint64))


def test_p2p_transport_single_rank_matches_combine():
    # the NVLink mailbox combine (csrc/xgpu.cu) at world 1: publish, wait, fold;
    # repeated calls alternate the epoch-parity buffers
    from paper_1401_6235_b200 import dist as D
    from paper_1401_6235_b200 import reduce as R

    tp = D.P2PTransport()
    rng = np.random.default_rng(4)
    for trial in range(5):
        n = 3 * 65536 + 17 * trial
        x = _t(rng.uniform(-1, 1, n) * np.exp2(rng.integers(-20, 21, n)))
        want = R.vtsum(x)
        part = torch.empty(2, dtype=torch.float64, device=DEV)
        R.vtsum(x, out=part)
        tp.combine(part, [n])
        assert (part[0].item(), part[1].item()) == (want.value, want.error)
        part32 = torch.empty(2, dtype=torch.float32, device=DEV)
        R.vtsum(x.float(), out=part32)
        w32 = R.vtsum(x.float())
        tp.combine(part32, [n])
        assert (part32[0].item(), part32[1].item()) == (w32.value, w32.error)
    assert tp.status() == 0


def test_p2p_fused_reduce_single_rank_matches_reduction():
    # tf_xgpu_reduce: the reduction and the mailbox exchange in ONE launch (the
    # last CTA publishes, waits and folds); at world 1 it must return exactly the
    # plain reduction, for every rop, both dtypes, unaligned views and n == 0,
    # interleaved with combine() calls (one shared epoch sequence)
    from paper_1401_6235_b200 import dist as D
    from paper_1401_6235_b200 import reduce as R

    tp = D.P2PTransport()
    tp2 = D.P2PTransport()  # a second transport in the same job reuses the mapping
    rng = np.random.default_rng(77)
    for trial, n in enumerate([5 * 65536, 3 * 131072 + 77, 1, 0, 65536 * 40 + 3]):
        for tdt in (torch.float64, torch.float32):
            x = _t(rng.uniform(-1, 1, n + 1) * np.exp2(rng.integers(-20, 21, n + 1))).to(tdt)
            y = _t(rng.uniform(-1, 1, n + 1)).to(tdt)
            for xs, ys in ((x[:n], y[:n]), (x[1:], y[1:])):  # aligned and unaligned
                for rop, planes, ref in (("sum", (xs,), lambda: R.vtsum(xs)),
                                         ("sum2", (xs, ys), lambda: R.vtsum2((xs, ys))),
                                         ("dot", (xs, ys), lambda: R.vtdot(xs, ys))):
                    want = ref()
                    got = (tp if trial % 2 else tp2).reduce(rop, planes, [n]).cpu().tolist()
                    assert (got[0], got[1]) == (want.value, want.error), (rop, n, tdt)
                    part = torch.tensor([want.value, want.error], dtype=tdt, device=DEV)
                    tp.combine(part, [n])
                    assert part.cpu().tolist() == [want.value, want.error]
    assert tp.status() == 0


def test_p2p_split_form_single_rank():
    # publish / collect (tf_xgpu_publish, tf_xgpu_reduce_publish, tf_xgpu_collect):
    # the same bits as the fused forms; one pending exchange at a time
    from paper_1401_6235_b200 import _lib
    from paper_1401_6235_b200 import dist as D
    from paper_1401_6235_b200 import reduce as R

    tp = D.P2PTransport()
    rng = np.random.default_rng(11)
    with pytest.raises(ValueError, match="no published exchange"):
        tp.collect(torch.empty(2, dtype=torch.float64, device=DEV))
    for trial, n in enumerate([3 * 65536 + 5, 0, 1, 70000]):
        x = _t(rng.uniform(-1, 1, n) * np.exp2(rng.integers(-20, 21, n)))
        y = _t(rng.uniform(-1, 1, n))
        for rop, planes, ref in (("sum", (x,), lambda: R.vtsum(x)),
                                 ("dot", (x, y), lambda: R.vtdot(x, y))):
            want = ref()
            o = tp.reduce(rop, planes, [n], publish_only=True)
            with pytest.raises(ValueError, match="awaits tf_xgpu_collect"):
                tp.combine(torch.zeros(2, dtype=torch.float64, device=DEV), [n])
            local = o.cpu().tolist()  # the local result, as published
            assert local == [want.value, want.error] or n == 0
            tp.collect(o)
            assert o.cpu().tolist() == [want.value, want.error], (rop, n)
        part = torch.tensor([want.value, want.error], device=DEV).float()
        tp.publish(part, [n])
        tp.collect(part)
        w32 = torch.tensor([want.value, want.error], device=DEV).float().cpu().tolist()
        assert part.cpu().tolist() == (w32 if n else [0.0, 0.0])
    assert tp.status() == 0
    assert _lib.lib().tf_xgpu_collect(_lib.TF_F64, None, None) != 0  # bad arguments


@pytest.mark.parametrize("world", [2, 3, 4, 7, 8, 16])
@pytest.mark.parametrize("rop", ["sum", "sum2", "dot"])
def test_p2p_fused_reduce_emulated_ranks_match_one_gpu(world, rop):
    # the fused reduce + exchange for `world` ranks as one grid on this GPU
    # (tf_xgpu_reduce_emulate): shards cut by dist.shard_tiles (complete
    # subtrees, trailing ranks possibly empty); every rank must end with the
    # one-GPU reduction's bits — shard invariance through the fused kernel
    import ctypes

    from paper_1401_6235_b200 import _lib
    from paper_1401_6235_b200 import dist as D
    from paper_1401_6235_b200 import reduce as R

    rng = np.random.default_rng(1000 + world)
    for tdt in (torch.float64, torch.float32):
        L = R.tile_elems(np.float64 if tdt == torch.float64 else np.float32)
        n = 9 * L + 12345
        x = _t(rng.uniform(-1, 1, n) * np.exp2(rng.integers(-25, 26, n))).to(tdt)
        y = _t(rng.uniform(-1, 1, n)).to(tdt)
        ref = {"sum": lambda: R.vtsum(x), "sum2": lambda: R.vtsum2((x, y)),
               "dot": lambda: R.vtdot(x, y)}[rop]()
        counts = D.shard_counts(n, world, L)
        outs = torch.empty((world, 2), dtype=tdt, device=DEV)
        c = (ctypes.c_int64 * world)(*counts)
        dt = _lib.TF_F64 if tdt == torch.float64 else _lib.TF_F32
        rc = _lib.lib().tf_xgpu_reduce_emulate(_lib.ROP_IDS[rop], dt, world, x.data_ptr(),
                                               None if rop == "sum" else y.data_ptr(), c,
                                               outs.data_ptr(),
                                               torch.cuda.current_stream().cuda_stream)
        _lib.check(rc, "tf_xgpu_reduce_emulate")
        for r, (v0, v1) in enumerate(outs.cpu().tolist()):
            assert (v0, v1) == (ref.value, ref.error), (world, rop, tdt, r, counts)


@pytest.mark.parametrize("world", [2, 3, 5, 8, 13, 64])
@pytest.mark.parametrize("tdt", [torch.float64, torch.float32])
def test_p2p_protocol_emulated_ranks_match_combine(world, tdt):
    # the multi-rank mailbox protocol of csrc/xgpu.cu (publish to every peer,
    # system fence, epoch flags, bounded wait, skip-tree fold) with every rank
    # played by one block of a single kernel on this GPU, over 6 epochs (both
    # parity buffers, each reused): every rank must end with exactly the
    # tf_combine result, empty shards skipped as tf_combine skips them
    import ctypes

    from paper_1401_6235_b200 import _lib
    from paper_1401_6235_b200 import reduce as R

    rng = np.random.default_rng(world)
    parts = []
    for r in range(world):
        x = _t(rng.uniform(-1, 1, 70000) * np.exp2(rng.integers(-30, 31, 70000))).to(tdt)
        p = torch.empty(2, dtype=tdt, device=DEV)
        R.vtsum(x, out=p)
        parts.append(p)
    P = torch.stack(parts)
    counts = [0 if (r % 4 == 1) else 70000 for r in range(world)]
    want = R.combine(P, counts)
    io = P.clone().contiguous()
    dt = _lib.TF_F64 if tdt == torch.float64 else _lib.TF_F32
    c = (ctypes.c_int64 * world)(*counts)
    stream = torch.cuda.current_stream().cuda_stream
    rc = _lib.lib().tf_xgpu_emulate(dt, world, io.data_ptr(), c, 6, stream)
    _lib.check(rc, "tf_xgpu_emulate")
    got = io.cpu().tolist()
    for r in range(world):
        assert (got[r][0], got[r][1]) == (want.value, want.error), (r, got[r], want)


def test_concurrent_threads_and_streams(oracle):
    # four Python threads, each on its own CUDA stream, run elementwise ops,
    # reductions (per-stream workspaces) and host-plane calls (per-device pipe
    # lock) at the same time; every result must still be bit-exact
    import threading

    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R

    n = (1 << 21) + 7
    errors = []

    def work(seed):
        try:
            rng = np.random.default_rng(seed)
            x = rng.uniform(-1, 1, n)
            y = rng.uniform(-1, 1, n)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                X, Y = _t(x), _t(y)
                for _ in range(3):
                    out = K.empty_twofold(n, torch.float64)
                    K.vtmul2(K.TwofoldArray(X, Y), K.TwofoldArray(Y, X), out)
                    z = R.vtdot(X, Y)
                    s.synchronize()
                    w = oracle.elementwise("vtmul2", x, y, y, x)
                    assert np.array_equal(out.value.cpu().numpy().view(np.uint64), w[0].view(np.uint64))
                    wd = oracle.reduce("dot", x, y, geometry=_geom(np.float64))
                    assert (z.value, z.error) == (float(wd[0]), float(wd[1]))
                    oh = K.empty_twofold(n, np.float64, device="cpu")
                    K.vtadd2(K.TwofoldArray(x, y), K.TwofoldArray(y, x), oh)
                    wa = oracle.elementwise("vtadd2", x, y, y, x)
                    assert np.array_equal(oh.value.view(np.uint64), wa[0].view(np.uint64))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("tdt", [torch.float64, torch.float32])
def test_reduce_pair_every_combination_matches_single(tdt):
    # tf_reduce_pair: two reductions in one pass; each result must be the single
    # reduction's bits — every (rop1, rop2), full and partial tiles, unaligned
    # views (scalar path), n = 1 and n = 0
    from paper_1401_6235_b200 import reduce as R

    rng = np.random.default_rng(17)
    single = {"vtsum": lambda x, y: R.vtsum(x), "vtsum2": lambda x, y: R.vtsum2((x, y)),
              "vtdot": lambda x, y: R.vtdot(x, y)}
    call = {"vtsum": lambda x, y: ("vtsum", x), "vtsum2": lambda x, y: ("vtsum2", (x, y)),
            "vtdot": lambda x, y: ("vtdot", x, y)}
    for n in (3 * 131072 + 4099, 65536 * 2, 1, 0):
        base_x = _t(rng.uniform(-1, 1, n + 1) * np.exp2(rng.integers(-30, 31, n + 1))).to(tdt)
        base_y = _t(rng.uniform(-1, 1, n + 1)).to(tdt)
        for x, y in ((base_x[:n], base_y[:n]), (base_x[1:], base_y[1:])):
            for r1 in single:
                for r2 in single:
                    got = R.batch([call[r1](x, y), call[r2](x, y)])
                    want = [single[r1](x, y), single[r2](x, y)]
                    assert [tuple(g) for g in got] == [tuple(w) for w in want], (n, r1, r2)


def test_reduce_batch_config4_ill_conditioned_and_routing(oracle):
    # config 4's step as one pass on an ill-conditioned dot; non-pairable calls
    # fall back to single launches; host planes route to host_batch
    from paper_1401_6235_b200 import reduce as R

    n = (1 << 21) + 77
    x, y = _ill_dot(n, 1e16, 11)
    X, Y = _t(x), _t(y)
    zd, zs = R.batch([("vtdot", X, Y), ("vtsum", X)])
    assert tuple(zd) == tuple(R.vtdot(X, Y)) and tuple(zs) == tuple(R.vtsum(X))
    w = oracle.reduce("dot", x, y, geometry=_geom(np.float64))
    assert tuple(zd) == (float(w[0]), float(w[1]))
    ok, err, s, t = oracle.bound_ok(zd.value, zd.error, "dot", x, y)
    assert ok
    Z = _t(np.ascontiguousarray(y[::-1]))
    got = R.batch([("vtsum", Y), ("vtdot", X, Y), ("vtsum", Z), ("vtsum", Z)])
    want = [R.vtsum(Y), R.vtdot(X, Y), R.vtsum(Z), R.vtsum(Z)]
    assert [tuple(g) for g in got] == [tuple(v) for v in want]
    out = torch.empty((2, 2), dtype=torch.float64, device=DEV)
    R.batch([("vtdot", X, Y), ("vtsum", X)], out=out)
    assert out.cpu().tolist() == [list(zd), list(zs)]
    hz = R.batch([("vtdot", x, y), ("vtsum", x)])
    assert [tuple(v) for v in hz] == [tuple(zd), tuple(zs)]
    with pytest.raises(ValueError, match="mix"):
        R.batch([("vtdot", X, Y), ("vtsum", X.float())])
    with pytest.raises(ValueError, match="unknown"):
        R.batch([("vtnope", X)])


def test_reduce_out_must_be_contiguous_and_on_the_planes_device():
    # a strided out view (t[:, 0]) would receive the wrong elements
    from paper_1401_6235_b200 import reduce as R

    x = torch.ones(1000, dtype=torch.float64, device=DEV)
    t = torch.zeros((2, 2), dtype=torch.float64, device=DEV)
    with pytest.raises(ValueError, match="contiguous"):
        R.vtsum(x, out=t[:, 0])
    with pytest.raises(ValueError, match="2-element"):
        R.vtsum(x, out=torch.zeros(2, dtype=torch.float64))
    out = torch.zeros(2, dtype=torch.float64, device=DEV)
    R.vtsum(x, out=out)
    assert out.tolist() == [1000.0, 0.0]


def test_captured_reduction_keeps_its_workspace_when_the_cache_grows(oracle):
    # a graph bakes in its workspace address; a later, larger eager
    # reduction on the same stream must not free it (use-after-free on replay),
    # and replays must not share a ticket counter with eager reductions
    from paper_1401_6235_b200 import reduce as R

    rng = np.random.default_rng(77)
    small = rng.uniform(-1, 1, 3 * 65536 + 5)
    big = rng.uniform(-1, 1, 64 * 65536 + 3)
    xs, xb = _t(small), _t(big)
    s = torch.cuda.Stream()
    out = torch.zeros(2, dtype=torch.float64, device=DEV)
    with torch.cuda.stream(s):
        R.vtsum(xs, out=out)  # warm the per-stream cache at the small size
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        R.vtsum(xs, out=out)
    with torch.cuda.stream(s):
        zb = R.vtsum(xb)  # grows the eager workspace of this stream
        junk = torch.full((1 << 22,), 3.0, dtype=torch.float64, device=DEV)  # reuse freed memory
    V, W, Kk = R.geometry(np.float64)
    want_s = oracle.reduce("sum", small, geometry=(V, W, Kk))
    want_b = oracle.reduce("sum", big, geometry=(V, W, Kk))
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert out.tolist() == [float(want_s[0]), float(want_s[1])]
    assert (zb.value, zb.error) == (float(want_b[0]), float(want_b[1]))
    del junk
