"""Past 2^31 elements: 64-bit indexing in every kernel family (B200, ~70 GB HBM).

Elementwise: vtadd (TwoSum) over 2^31+5 f32 elements checked on the device
against TwoSum evaluated with plain torch ops (each an IEEE-RN kernel, no
contraction), and the twofold sum of the same plane bit-exact against the oracle.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.fullsize]

N = (1 << 31) + 5


def test_elementwise_and_reduction_past_2g_elements(oracle):
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R
    from paper_1401_6235_b200 import workloads as W

    free, _ = torch.cuda.mem_get_info()
    if free < 80e9:
        pytest.skip("needs ~80 GB of free HBM")
    x = W.fill(torch.empty(N, dtype=torch.float32, device="cuda"), W.LOGU_SIGNED, 11, 0, -20.0, 20.0)
    y = W.fill(torch.empty(N, dtype=torch.float32, device="cuda"), W.LOGU_SIGNED, 12, 0, -20.0, 20.0)
    z = K.empty_twofold(N, torch.float32, K.CoupledArray)
    K.vtadd(x, y, z)
    s = x + y
    assert torch.equal(z.value, s)
    bv = s - x
    av = s - bv
    t = (x - av) + (y - bv)
    del s, bv, av
    assert torch.equal(z.error, t)
    del t, z, y
    torch.cuda.empty_cache()
    zs = R.vtsum(x)
    xh = x.cpu().numpy()
    w = oracle.reduce("sum", xh, geometry=R.geometry(np.float32))
    assert (zs.value, zs.error) == (float(w[0]), float(w[1]))


def test_device_batch_past_2g_elements():
    # the device batch (one launch, two ops over one shared plane) past 2^31
    # elements: vtmul (TwoProd) and vtsqrt checked against one launch per op on
    # a 1/1024 sample of positions spread over the whole index range
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import workloads as W

    free, _ = torch.cuda.mem_get_info()
    if free < 60e9:
        pytest.skip("needs ~60 GB of free HBM")
    x = W.fill(torch.empty(N, dtype=torch.float32, device="cuda"), W.LOGU_POS, 21, 0, -20.0, 20.0)
    a = K.empty_twofold(N, torch.float32, K.CoupledArray)
    b = K.empty_twofold(N, torch.float32, K.CoupledArray)
    K.batch([("vtmul", x, x, a), ("vtsqrt", x, b)])
    idx = torch.arange(0, N, 1021, device="cuda")
    idx = torch.cat([idx, torch.tensor([N - 1], device="cuda")])
    xs = x[idx].contiguous()
    del x
    torch.cuda.empty_cache()
    wa = K.empty_twofold(xs.numel(), torch.float32, K.CoupledArray)
    wb = K.empty_twofold(xs.numel(), torch.float32, K.CoupledArray)
    K.vtmul(xs, xs, wa)
    K.vtsqrt(xs, wb)
    assert torch.equal(a.value[idx], wa.value) and torch.equal(a.error[idx], wa.error)
    assert torch.equal(b.value[idx], wb.value) and torch.equal(b.error[idx], wb.error)


def test_reduce_pair_past_2g_elements():
    # the one-pass dot + sum (tf_reduce_pair) past 2^31 elements: bit-identical
    # to the two single reductions (64-bit tile and element indexing)
    from paper_1401_6235_b200 import reduce as R
    from paper_1401_6235_b200 import workloads as W

    free, _ = torch.cuda.mem_get_info()
    if free < 40e9:
        pytest.skip("needs ~40 GB of free HBM")
    x = W.fill(torch.empty(N, dtype=torch.float32, device="cuda"), W.LOGU_SIGNED, 31, 0, -20.0, 20.0)
    y = W.fill(torch.empty(N, dtype=torch.float32, device="cuda"), W.UNIFORM, 32, 0, -1.0, 1.0)
    zd, zs = R.batch([("vtdot", x, y), ("vtsum", x)])
    assert tuple(zd) == tuple(R.vtdot(x, y))
    assert tuple(zs) == tuple(R.vtsum(x))
