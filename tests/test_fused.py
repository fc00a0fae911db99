"""Fused demo chains (demos.py:153-238) over batches: the oracle and the GPU
kernels reproduce the reference-generated fixtures bit for bit, and the
reference's own transcript tokens for the quadratic and Gauss demo cases
(goldens quad_*.txt / gauss_*.txt) render identically from the GPU results."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

FU = np.load(GOLDEN / "fused.npz")
META = json.loads((GOLDEN / "fused.json").read_text())


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    if a.shape != b.shape or not np.array_equal(na, nb):
        return False
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return np.array_equal(a[~na].view(u), b[~nb].view(u))


def _fmt(v, e):
    def g(x):
        x = float(x)
        return "nan" if x != x else "%.*g" % (6, x)
    return "%s[%s]" % (g(v), g(e))


FMTS = ["f64", "f32"]


@pytest.mark.parametrize("fmt", FMTS)
def test_oracle_axpy_submul(oracle, fmt):
    ins = [FU["axpy/%s/in%d" % (fmt, k)] for k in range(6)]
    z = oracle.fused("axpy", *ins)
    assert bits_equal(np.stack(z), FU["axpy/%s/out" % fmt])
    z = oracle.fused("submul", *ins)
    assert bits_equal(np.stack(z), FU["submul/%s/out" % fmt])


@pytest.mark.parametrize("fmt", FMTS)
def test_oracle_quadratic(oracle, fmt):
    ins = [FU["quad/%s/in%d" % (fmt, k)] for k in range(6)]
    outs = oracle.fused("quadratic", *ins)
    for k in range(6):
        assert bits_equal(outs[k], FU["quad/%s/out%d" % (fmt, k)]), k


@pytest.mark.parametrize("fmt", FMTS)
def test_oracle_gauss3(oracle, fmt):
    g = lambda k: FU["gauss3/%s/%s" % (fmt, k)]  # noqa: E731
    xv, xe = oracle.fused("gauss3", g("Av").reshape(-1), g("Ae").reshape(-1),
                          g("Fv").reshape(-1), g("Fe").reshape(-1))
    assert bits_equal(xv.reshape(3, -1), g("Xv")) and bits_equal(xe.reshape(3, -1), g("Xe"))


def _cuda(a):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", FMTS)
def test_gpu_axpy_submul(fmt):
    from paper_1401_6235_b200 import fused as F
    from paper_1401_6235_b200.kernels import TwofoldArray as TA

    ins = [_cuda(FU["axpy/%s/in%d" % (fmt, k)]) for k in range(6)]
    a, x, y = TA(ins[0], ins[1]), TA(ins[2], ins[3]), TA(ins[4], ins[5])
    z = F.vtaxpy(a, x, y)
    assert bits_equal(np.stack([z.value.cpu().numpy(), z.error.cpu().numpy()]),
                      FU["axpy/%s/out" % fmt])
    z = F.vtsubmul(a, x, y)
    assert bits_equal(np.stack([z.value.cpu().numpy(), z.error.cpu().numpy()]),
                      FU["submul/%s/out" % fmt])


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", FMTS)
def test_gpu_quadratic_and_reference_transcripts(fmt):
    from paper_1401_6235_b200 import fused as F
    from paper_1401_6235_b200.kernels import TwofoldArray as TA

    ins = [_cuda(FU["quad/%s/in%d" % (fmt, k)]) for k in range(6)]
    d, x0, x1 = F.vtquadratic(TA(ins[0], ins[1]), TA(ins[2], ins[3]), TA(ins[4], ins[5]))
    outs = [t.cpu().numpy() for z in (d, x0, x1) for t in z]
    for k in range(6):
        assert bits_equal(outs[k], FU["quad/%s/out%d" % (fmt, k)]), k
    for i, tok in enumerate(META["quad/%s" % fmt]["tokens"]):
        assert _fmt(outs[0][i], outs[1][i]) == tok["d"]
        assert _fmt(outs[2][i], outs[3][i]) == tok["x0"]
        assert _fmt(outs[4][i], outs[5][i]) == tok["x1"]


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", FMTS)
def test_gpu_gauss3_and_reference_transcripts(fmt):
    from paper_1401_6235_b200 import fused as F
    from paper_1401_6235_b200.kernels import TwofoldArray as TA

    g = lambda k: FU["gauss3/%s/%s" % (fmt, k)]  # noqa: E731
    x = F.vtgauss3(TA(_cuda(g("Av")), _cuda(g("Ae"))), TA(_cuda(g("Fv")), _cuda(g("Fe"))))
    xv, xe = x.value.cpu().numpy(), x.error.cpu().numpy()
    assert bits_equal(xv, g("Xv")) and bits_equal(xe, g("Xe"))
    for s, case in enumerate(("well3", "ill3")):
        got = [_fmt(xv[r, s], xe[r, s]) for r in range(3)]
        assert got == META["gauss3/%s" % fmt]["tokens"][case], (case, got)


@pytest.mark.gpu
def test_gpu_fused_large_matches_composition():
    import torch

    from paper_1401_6235_b200 import fused as F
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import workloads as W

    n = (1 << 22) + 3
    ps = W.PlaneSet("config2", n, torch.float64, 0)
    x0, x1, y0, y1 = ps.planes("vtadd2")
    a = K.TwofoldArray(*ps.planes("vtsqrt1"))
    t = K.empty_twofold(n, torch.float64)
    K.vtmul2(a, K.TwofoldArray(x0, x1), t)
    want = K.empty_twofold(n, torch.float64)
    K.vtadd2(t, K.TwofoldArray(y0, y1), want)
    z = F.vtaxpy(a, K.TwofoldArray(x0, x1), K.TwofoldArray(y0, y1))
    assert torch.equal(z.value, want.value) and torch.equal(z.error, want.error)


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("offset", [1, 2])
def test_gpu_fused_misaligned_and_tails_match_aligned(fmt, offset):
    # the vector body needs every plane aligned to the vector width; shifted
    # views take the scalar path, odd n leaves a scalar tail — bits unchanged
    import torch

    from paper_1401_6235_b200 import fused as F
    from paper_1401_6235_b200.kernels import TwofoldArray as TA

    dt = torch.float64 if fmt == "f64" else torch.float32
    n = 4099
    rng = np.random.default_rng(3)
    base = [rng.uniform(0.5, 2.0, n + offset) for _ in range(6)]
    base[4] *= 0.1  # c small: real roots for the quadratic

    mis = [torch.as_tensor(b, dtype=dt, device="cuda")[offset:offset + n] for b in base]
    al = [m.clone() for m in mis]  # the same values in fresh (aligned) allocations
    for fn in (F.vtaxpy, F.vtsubmul):
        za = fn(TA(al[0], al[1]), TA(al[2], al[3]), TA(al[4], al[5]))
        zm = fn(TA(mis[0], mis[1]), TA(mis[2], mis[3]), TA(mis[4], mis[5]))
        assert torch.equal(za.value, zm.value) and torch.equal(za.error, zm.error)
    qa = F.vtquadratic(TA(al[0], al[1]), TA(al[2], al[3]), TA(al[4], al[5]))
    qm = F.vtquadratic(TA(mis[0], mis[1]), TA(mis[2], mis[3]), TA(mis[4], mis[5]))
    for a, m in zip(qa, qm):
        assert bits_equal(np.stack([a.value.cpu().numpy(), a.error.cpu().numpy()]),
                          np.stack([m.value.cpu().numpy(), m.error.cpu().numpy()]))
