"""B200-native data-parallel core of twofold arithmetic (Latkin, arXiv 1401.6235).

Drop-in for the reference's batch-kernel layer ``twofold.kernels``
(/root/reference/pkg/src/twofold/kernels.py): the same names and contracts,
with planes as CUDA tensors (or numpy arrays, staged through the device), every
kernel a hand-written sm_100a CUDA kernel behind the C ABI in
include/twofold_b200.h.  Adds twofold reductions, Horner and multi-GPU sharding.
"""

from . import kernels  # noqa: F401
from . import dist, fused, interleaved, reduce, workloads  # noqa: F401
from .kernels import KERNELS, CoupledArray, KernelSpec, TwofoldArray, empty_twofold  # noqa: F401
from .reduce import Twofold, vtdot, vthorner, vtsum, vtsum2  # noqa: F401

__version__ = "0.1.0"

__all__ = ["kernels", "interleaved", "fused", "reduce", "dist", "workloads", "KERNELS", "KernelSpec", "TwofoldArray", "CoupledArray",
           "empty_twofold", "Twofold", "vtsum", "vtsum2", "vtdot", "vthorner",
           "__version__"]
