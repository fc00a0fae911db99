"""Interleaved (AoS) layout: same bits as the split layout and the reference
goldens, for every op and both dtypes; conversions round-trip exactly."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import GOLDEN  # noqa: E402

ELEM = np.load(GOLDEN / "elementwise.npz")
NAMES = sorted({k.split("/")[0] for k in ELEM.files})
ARITY = {}


def _arity(name):
    from paper_1401_6235_b200 import kernels as K

    if name == "div_rem":
        return "11"
    if name == "sqrt_resid":
        return "u1"
    return K.KERNELS[name].arity


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    if a.shape != b.shape or not np.array_equal(na, nb):
        return False
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return np.array_equal(a[~na].view(u), b[~nb].view(u))


def _pairs(v, e, offset=0):
    dt = torch.float64 if v.dtype == np.float64 else torch.float32
    host = np.stack([v, e], axis=1)
    if offset == 0:
        return torch.from_numpy(np.ascontiguousarray(host)).cuda()
    buf = torch.empty(host.size + offset, dtype=dt, device="cuda")
    view = buf[offset:].view(-1, 2)
    view.copy_(torch.from_numpy(host))
    return view


def _plane(v, offset=0):
    if offset == 0:
        return torch.from_numpy(np.ascontiguousarray(v)).cuda()
    dt = torch.float64 if v.dtype == np.float64 else torch.float32
    buf = torch.empty(v.shape[0] + offset, dtype=dt, device="cuda")
    buf[offset:].copy_(torch.from_numpy(v))
    return buf[offset:]


def _run(name, fmt, offset=0):
    from paper_1401_6235_b200 import interleaved as IL

    ar = _arity(name)
    ins = []
    k = 0
    while "%s/%s/in%d" % (name, fmt, k) in ELEM.files:
        ins.append(ELEM["%s/%s/in%d" % (name, fmt, k)])
        k += 1
    n = ins[0].shape[0]
    dt = torch.float64 if fmt == "f64" else torch.float32
    if ar == "22":
        args = (_pairs(ins[0], ins[1], offset), _pairs(ins[2], ins[3], offset))
    elif ar == "21":
        args = (_pairs(ins[0], ins[1], offset), _plane(ins[2], offset))
    elif ar == "11":
        args = (_plane(ins[0], offset), _plane(ins[1], offset))
    elif ar == "u2":
        args = (_pairs(ins[0], ins[1], offset),)
    else:
        args = (_plane(ins[0], offset),)
    if offset:
        buf = torch.full((2 * n + offset,), 7.0, dtype=dt, device="cuda")
        out = buf[offset:].view(-1, 2)
    else:
        out = torch.full((n, 2), 7.0, dtype=dt, device="cuda")
    IL.KERNELS[name](*args, out)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    return o[:, 0].copy(), o[:, 1].copy()


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["f64", "f32"])
@pytest.mark.parametrize("name", NAMES)
def test_interleaved_matches_reference_golden(name, fmt):
    for offset in (0, 1):
        r0, r1 = _run(name, fmt, offset)
        assert bits_equal(r0, ELEM["%s/%s/out0" % (name, fmt)]), (name, offset)
        assert bits_equal(r1, ELEM["%s/%s/out1" % (name, fmt)]), (name, offset)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_conversions_round_trip(dtype):
    from paper_1401_6235_b200 import interleaved as IL
    from paper_1401_6235_b200 import kernels as K

    for n in (0, 1, 7, 1 << 20 | 3):
        v = torch.randn(n, dtype=dtype, device="cuda")
        e = torch.randn(n, dtype=dtype, device="cuda") * 1e-17
        p = IL.from_split(K.TwofoldArray(v, e))
        assert torch.equal(p[:, 0], v) and torch.equal(p[:, 1], e)
        back = IL.to_split(p)
        assert torch.equal(back.value, v) and torch.equal(back.error, e)


_CONV_SWEEP = r"""
import torch
from paper_1401_6235_b200 import interleaved as IL, kernels as K
for dtype in (torch.float64, torch.float32):
    E = 32 // torch.empty(0, dtype=dtype).element_size()
    sizes = sorted({1, E - 1, E, E + 1, 2 * E + 1, 255 * E, 256 * E, 512 * E - 1, 512 * E,
                    512 * E + 1, 1024 * E + E // 2, (1 << 21) + 5})
    for n in sizes:
        for off in (0, 1, 4):  # views off the 32-byte alignment take the 16-byte / scalar kernels
            vb = torch.randn(n + off, dtype=dtype, device="cuda")
            eb = torch.randn(n + off, dtype=dtype, device="cuda")
            v, e = vb[off:], eb[off:]
            G = E // 2  # guard rows: E/2 pairs = 32 bytes, so an aligned base stays aligned
            guard = torch.full((n + 2 * G, 2), 7.0, dtype=dtype, device="cuda")
            p = guard[G:n + G]
            IL.from_split(K.TwofoldArray(v, e), p)
            assert torch.equal(p[:, 0], v) and torch.equal(p[:, 1], e), (dtype, n, off)
            assert (guard[:G] == 7).all() and (guard[n + G:] == 7).all(), (dtype, n, off)
            ob = [torch.full((n + off + 2 * E,), 7.0, dtype=dtype, device="cuda") for _ in range(2)]
            o = K.TwofoldArray(ob[0][off + E:off + E + n], ob[1][off + E:off + E + n])
            IL.to_split(p, o)
            assert torch.equal(o.value, v) and torch.equal(o.error, e), (dtype, n, off)
            for b in ob:
                assert (b[:off + E] == 7).all() and (b[off + E + n:] == 7).all(), (dtype, n, off)
print("conv-ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("lean", ["1", "0", None])
def test_conversions_sweep_both_variants(lean):
    # lean 32-byte step kernels (default) and the 16-byte grid-stride kernels
    # (TF_CONV_LEAN=0): sizes around the vector and CTA boundaries, aligned and
    # misaligned views, guard elements either side of every destination
    import os, subprocess, sys
    env = dict(os.environ)
    env.pop("TF_CONV_LEAN", None)
    if lean is not None:
        env["TF_CONV_LEAN"] = lean
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CONV_SWEEP], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "conv-ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_interleaved_large_matches_split():
    from paper_1401_6235_b200 import interleaved as IL
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import workloads as W

    # odd lengths: the n % E remainder takes the lean kernel's masked step
    for cfg, n, dt, names in (("config2", (1 << 22) + 1, torch.float64, ("vtadd2", "vtdiv2", "vtsqrt1")),
                              ("config3", (1 << 22) + 3, torch.float32, ("vtadd2", "vtmul2", "vtdiv2"))):
        ps = W.PlaneSet(cfg, n, dt, 0)
        for name in names:
            planes = ps.planes(name)
            out = K.empty_twofold(n, dt)
            K.KERNELS[name].loop(*planes, *out)
            x = IL.from_split(K.TwofoldArray(planes[0], planes[1]))
            args = (x,) if name == "vtsqrt1" else (x, IL.from_split(K.TwofoldArray(planes[2], planes[3])))
            po = IL.empty_pairs(n, dt)
            IL.KERNELS[name](*args, po)
            assert torch.equal(po[:, 0], out.value) and torch.equal(po[:, 1], out.error), (name, dt)


def test_interleaved_validation_without_gpu():
    from paper_1401_6235_b200 import interleaved as IL

    x = torch.zeros((8, 2), dtype=torch.float64)
    with pytest.raises(ValueError, match="CUDA tensors"):
        IL.vtadd2(x, x, x)
    with pytest.raises(ValueError, match="CUDA tensors"):
        IL.vtadd2(np.zeros((8, 2)), x, x)


@pytest.mark.gpu
def test_conversions_validate_before_launch():
    # a short or float32 out, a 1-D pair array or aliasing planes
    # raise ValueError instead of reaching the kernel with raw pointers
    from paper_1401_6235_b200 import interleaved as IL
    from paper_1401_6235_b200 import kernels as K

    v = torch.ones(64, dtype=torch.float64, device="cuda")
    e = torch.zeros(64, dtype=torch.float64, device="cuda")
    x = K.TwofoldArray(v, e)
    with pytest.raises(ValueError, match="lengths differ"):
        IL.from_split(x, torch.empty((32, 2), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="mix"):
        IL.from_split(x, torch.empty((64, 2), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError, match="pair arrays"):
        IL.from_split(x, torch.empty(128, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="lengths differ"):
        IL.from_split(K.TwofoldArray(v, e[:10]))
    buf = torch.empty(256, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="alias"):
        IL.from_split(K.TwofoldArray(buf[:64], e), buf[:128].view(64, 2))
    p = IL.from_split(x)
    with pytest.raises(ValueError, match="pair arrays"):
        IL.to_split(p.reshape(-1))
    with pytest.raises(ValueError, match="lengths differ"):
        IL.to_split(p, K.TwofoldArray(torch.empty(10, dtype=torch.float64, device="cuda"),
                                      torch.empty(64, dtype=torch.float64, device="cuda")))
    with pytest.raises(ValueError, match="overlap"):
        same = torch.empty(64, dtype=torch.float64, device="cuda")
        IL.to_split(p, K.TwofoldArray(same, same))
    back = IL.to_split(p)
    assert torch.equal(back.value, v) and torch.equal(back.error, e)
