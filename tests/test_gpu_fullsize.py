"""Parity at BASELINE.json's full sizes (B200).

Every element of every output plane is compared bit-exactly with the oracle:
config 2 (f64 x5 ops, n=2^28), config 3 (f32 x3 ops, n=2^30), config 4 (dot and
sum of its own plane, n=2^30, cond 1e16: bit-exact in the canonical order —
against the live oracle and the committed golden — and inside the 4u·Σ|terms|
bound against the exact accumulator) and config 5 (Horner, 2^26
points, plus the cancellation flag).  Inputs are the bench's own device-
generated planes (paper_1401_6235_b200.workloads), copied to the host.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.fullsize]


def _host(t):
    return t.cpu().numpy()


def _bits_equal_chunked(a, b, chunk=1 << 26):
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    for i in range(0, a.shape[0], chunk):
        x, y = a[i:i + chunk], b[i:i + chunk]
        nx, ny = np.isnan(x), np.isnan(y)
        if not np.array_equal(nx, ny):
            return False
        if not np.array_equal(x.view(u)[~nx], y.view(u)[~ny]):
            return False
    return True


def _run_config(oracle, config, names, n, dtype):
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import workloads as W

    ps = W.PlaneSet(config, n, dtype, 0)
    out = K.empty_twofold(n, dtype)
    npdt = np.float64 if dtype == torch.float64 else np.float32
    ref = (np.empty(n, npdt), np.empty(n, npdt))
    for name in names:
        planes = ps.planes(name)
        K.KERNELS[name].loop(*planes, out.value, out.error)
        torch.cuda.synchronize()
        ins = [_host(p) for p in planes]
        oracle.elementwise(name, *ins, out=ref)
        z0, z1 = _host(out.value), _host(out.error)
        assert _bits_equal_chunked(z0, ref[0]), (config, name, "value plane")
        assert _bits_equal_chunked(z1, ref[1]), (config, name, "error plane")
        del ins, z0, z1


def test_config2_full_size_bit_exact(oracle):
    _run_config(oracle, "config2", ["vtadd2", "vtsub2", "vtmul2", "vtdiv2", "vtsqrt1"],
                1 << 28, torch.float64)


def test_config3_full_size_bit_exact(oracle):
    _run_config(oracle, "config3", ["vtadd2", "vtmul2", "vtdiv2"], 1 << 30, torch.float32)


def test_config1_bit_exact(oracle):
    _run_config(oracle, "config1", ["vtadd2", "vtmul2"], 1 << 20, torch.float64)


def test_config4_full_size_dot_and_sum(oracle):
    # BASELINE configs[3] as stated: the dot x.y AND the sum of its own plane p,
    # n = 2^30, cond ~1e16, half the terms with random exponents in [-50, 50]
    # (blocked ORO-style generator, run on the device as the bench does)
    import json

    from conftest import GOLDEN
    from paper_1401_6235_b200 import reduce as R
    from paper_1401_6235_b200 import workloads as W

    n = 1 << 30
    X, Y, P = W.config4_planes(n, 0, n, "cuda")
    zd, zs = R.vtdot(X, Y), R.vtsum(P)
    x, y, p = _host(X), _host(Y), _host(P)
    del X, Y, P
    geom = R.geometry(np.float64)
    golden = json.loads((GOLDEN / "config4.json").read_text())["prefixes"][str(n)]
    for name, z, rop, planes in (("vtdot", zd, "dot", (x, y)), ("vtsum", zs, "sum", (p,))):
        # bit-exact against the oracle's canonical order, live and as committed
        w = oracle.reduce(rop, *planes, geometry=geom)
        assert (z.value, z.error) == (float(w[0]), float(w[1])), name
        assert [z.value.hex(), z.error.hex()] == [golden[name]["z0"], golden[name]["z1"]], name
        # inside 4u * sum|terms| of the exact accumulator, at the stated condition
        ok, err, s, t = oracle.bound_ok(z.value, z.error, rop, *planes)
        assert ok, (name, float(err), float(t))
        cond = float((2 if rop == "dot" else 1) * t / abs(s))
        assert 0.5e16 < cond < 2e16, (name, cond)
        # the plain result in the same order is far off; the twofold is not
        rel_plain = abs(z.value - float(s)) / abs(float(s))
        rel_tf = float(err / abs(s))
        assert rel_tf < 1e-14 < rel_plain, (name, rel_tf, rel_plain)


def test_config5_full_size_horner(oracle):
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R
    from paper_1401_6235_b200 import workloads as W

    n = 1 << 26
    x = W.fill(torch.empty(n, dtype=torch.float64, device="cuda"), W.UNIFORM, 555, 0, 0.9, 1.1)
    out = K.empty_twofold(n, torch.float64)
    c = R.binomial_coeffs(20)
    R.vthorner(c, x, out)
    torch.cuda.synchronize()
    xh = _host(x)
    w0, w1 = oracle.horner(c, xh)
    z0, z1 = _host(out.value), _host(out.error)
    assert _bits_equal_chunked(z0, w0) and _bits_equal_chunked(z1, w1)
    nz = z0 != 0
    assert (np.abs(z1[nz]) >= 0.5 * np.abs(z0[nz])).mean() > 0.99
