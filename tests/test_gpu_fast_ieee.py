"""The branch-free f64 division / square-root fast paths (csrc/tf_math.cuh
div_fast, sqrt_fast) that the elementwise kernels run before falling back to
__ddiv_rn / __dsqrt_rn: wherever a fast path reports itself valid, its bits must
equal the intrinsic's.  tf_fastpath_check draws operands from every exponent
class (raw bit patterns with NaN/inf/subnormals, full-range exponents, the edges
of ptxas's range checks, hard-rounding mantissas)."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2, 3, 1401])
def test_fast_paths_match_intrinsics(seed):
    torch = pytest.importorskip("torch")
    assert torch.cuda.is_available()
    from paper_1401_6235_b200 import _lib

    counts = (ctypes.c_int64 * 4)()
    n = 1 << 28
    _lib.check(_lib.lib().tf_fastpath_check(0, n, seed, counts), "tf_fastpath_check")
    sqrt_ok, sqrt_bad, div_ok, div_bad = list(counts)
    assert sqrt_bad == 0 and div_bad == 0, list(counts)
    # the fast paths must actually cover most operands of the ordinary classes
    assert sqrt_ok > n // 8 and div_ok > n // 4, list(counts)
