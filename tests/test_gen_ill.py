"""The config-4 input generator (csrc/gen_ill.cu, blocked Ogita-Rump-Oishi
style): CPU checks of the host side — the condition numbers it promises, block
independence (any rank slice equals the same elements of the whole problem),
argument validation — and, on the GPU, that the device generator writes the
host generator's bits."""

import numpy as np
import pytest

from paper_1401_6235_b200 import _lib
from paper_1401_6235_b200 import workloads as W

B = W.GEN_BLOCK


def _host(kind, n_total, first, count, cond=1e16, emin=-50, emax=50, seed=4242):
    x, y = np.empty(count), np.empty(count)
    rc = _lib.lib().tf_gen_ill_host(kind, n_total, first, count, cond, seed, emin, emax,
                                    x.ctypes.data, y.ctypes.data if kind == 0 else None, 0)
    assert rc == 0, _lib.last_error()
    return x, y


@pytest.mark.parametrize("cond", [1e8, 1e16, 1e24])
@pytest.mark.parametrize("n", [1000, B, 3 * B + 12345])
def test_condition_numbers_as_requested(oracle, n, cond):
    x, y = _host(0, n, 0, n, cond)
    p, _ = _host(1, n, 0, n, cond)
    s, t = oracle.exact("dot", x, y)
    assert 2 * t / abs(s) == pytest.approx(cond, rel=1e-3)
    s, t = oracle.exact("sum", p)
    assert t / abs(s) == pytest.approx(cond, rel=1e-3)


def test_first_half_exponents_span_the_stated_range():
    # BASELINE: "half the pairs have random exponents in [-50, 50]"
    x, y = _host(0, B, 0, B)
    h = B // 2
    ex = np.frexp(x[:h])[1] - 1  # floor(log2|x|): mantissa U(-1, 1) times 2^e, e in [-50, 50]
    ey = np.frexp(y[:h])[1] - 1
    assert ex.min() < -45 and ex.max() == 49 and ey.min() < -45 and ey.max() == 49


def test_rank_slices_equal_the_whole_problem():
    n = 8 * B + 777
    x, y = _host(0, n, 0, n)
    p, _ = _host(1, n, 0, n)
    for first, count in ((0, 2 * B), (2 * B, 3 * B), (5 * B, n - 5 * B), (8 * B, 777)):
        xs, ys = _host(0, n, first, count)
        ps, _ = _host(1, n, first, count)
        assert np.array_equal(xs.view(np.uint64), x[first:first + count].view(np.uint64))
        assert np.array_equal(ys.view(np.uint64), y[first:first + count].view(np.uint64))
        assert np.array_equal(ps.view(np.uint64), p[first:first + count].view(np.uint64))
    # a prefix of whole blocks is the smaller problem itself
    x2, y2 = _host(0, 4 * B, 0, 4 * B)
    assert np.array_equal(x2.view(np.uint64), x[:4 * B].view(np.uint64))


def test_validation():
    L = _lib.lib()
    a = np.empty(10)
    assert L.tf_gen_ill_host(2, 10, 0, 10, 1e16, 1, -50, 50, a.ctypes.data, None, 0) == _lib.TF_EINVAL
    assert L.tf_gen_ill_host(1, 10, 5, 5, 1e16, 1, -50, 50, a.ctypes.data, None, 0) == _lib.TF_EINVAL
    assert "whole blocks" in _lib.last_error()
    assert L.tf_gen_ill_host(1, 10, 0, 11, 1e16, 1, -50, 50, a.ctypes.data, None, 0) == _lib.TF_EINVAL
    assert L.tf_gen_ill_host(1, 10, 0, 10, 0.5, 1, -50, 50, a.ctypes.data, None, 0) == _lib.TF_EINVAL
    assert L.tf_gen_ill_host(0, 10, 0, 10, 1e16, 1, -50, 50, a.ctypes.data, None, 0) == _lib.TF_EINVAL
    assert L.tf_gen_ill_host(1, 10, 0, 10, 1e16, 1, 50, -50, a.ctypes.data, None, 0) == _lib.TF_EINVAL
    assert L.tf_gen_ill_host(1, 0, 0, 0, 1e16, 1, -50, 50, None, None, 0) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("n,first,count", [(1 << 22, 0, 1 << 22), (5 * B + 99, 2 * B, 3 * B + 99),
                                           (1000, 0, 1000)])
def test_device_generator_writes_the_host_bits(n, first, count):
    torch = pytest.importorskip("torch")
    for kind in (0, 1):
        X = torch.empty(count, dtype=torch.float64, device="cuda")
        Y = torch.empty(count, dtype=torch.float64, device="cuda") if kind == 0 else None
        W.gen_ill(kind, X, Y, n_total=n, first=first)
        x, y = _host(kind, n, first, count)
        assert np.array_equal(X.cpu().numpy().view(np.uint64), x.view(np.uint64)), kind
        if kind == 0:
            assert np.array_equal(Y.cpu().numpy().view(np.uint64), y.view(np.uint64))
