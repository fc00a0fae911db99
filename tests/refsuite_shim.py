"""pytest plugin: run the reference's OWN test modules against the drop-in.

    PYTHONPATH=<repo>:<repo>/baseline/_ref NUMBA_CACHE_DIR=/tmp/nb \\
        python -m pytest -p tests.refsuite_shim -c /dev/null \\
        --rootdir baseline/_ref/twofold_tests baseline/_ref/twofold_tests/test_kernels.py ...

The reference package (``twofold``, staged unmodified into baseline/_ref by
tools/stage_reference.sh) is imported, then its array module ``twofold.kernels``
(/root/reference/pkg/src/twofold/kernels.py) is replaced by this repo's
drop-in, ``paper_1401_6235_b200.kernels``: every ``tf.kernels.vtXXX(numpy...)``
call in the reference's tests runs on the B200 through the host pipeline
(tf_elementwise_host).  The reference's scalar API (numba) stays in place — it
is what those tests compare the kernels against.

What the shim adapts (each a documented deviation of the drop-in, not of the
tests):
* ``KernelSpec.core``: the drop-in's core is a device op id (there is no
  host-callable core on a GPU path); criterion 10 calls ``spec.core(...)`` as
  its scalar oracle (test_acceptance.py:444-467), so the shim's registry
  carries the reference's numba core there.  ``func`` and ``loop`` are ours.
* ``_loop11(_div_rem)`` / ``_loop1u(_sqrt_resid)`` (test_acceptance.py:42-43):
  the loop factories map the reference's raw cores to the device's raw
  exact-transform loops (kernels.raw_loop), and a registry core to its
  kernel's raw launcher.
* gmpy2 is absent from this image: a stub module provides ``mpq`` as
  ``fractions.Fraction`` (exact rationals; criteria 4 and 7 use nothing else).
  ``mpfr`` / ``ieee`` raise if called (criteria 3 and 6 need them; they test the
  scalar API, not the kernels, and are not run).
"""

from __future__ import annotations

import fractions
import sys
import types


def _gmpy2_stub():
    g = types.ModuleType("gmpy2")
    g.mpq = fractions.Fraction

    class _Ctx:
        def __init__(self, *a):
            pass

        def __enter__(self):
            return self

        def __exit__(self, *a):
            return False

    def mpfr(*a, **k):
        raise NotImplementedError("gmpy2.mpfr is not available (stub): high-precision tests "
                                  "are out of the drop-in's scope")

    g.ieee = _Ctx
    g.context = _Ctx
    g.local_context = _Ctx
    g.mpfr = mpfr
    g.__stub__ = True
    return g


def install():
    if "gmpy2" not in sys.modules:
        try:
            import gmpy2  # noqa: F401
        except ImportError:
            sys.modules["gmpy2"] = _gmpy2_stub()

    import twofold  # the reference package (baseline/_ref)
    from twofold import arith as ref_arith
    from twofold import fp_core as ref_fp
    from twofold import kernels as ref_kernels

    from paper_1401_6235_b200 import kernels as ours

    shim = types.ModuleType("twofold.kernels")
    shim.__doc__ = ours.__doc__
    shim.__file__ = ours.__file__
    for name in ("TwofoldArray", "CoupledArray", "KernelSpec", "empty_twofold", "host_batch",
                 "batch", "raw_loop", "RAW_OPS"):
        setattr(shim, name, getattr(ours, name))
    ref_core_of = {name: spec.core for name, spec in ref_kernels.KERNELS.items()}
    registry = {}
    for name, spec in ours.KERNELS.items():
        registry[name] = spec._replace(core=ref_core_of[name])
        setattr(shim, name, spec.func)
    shim.KERNELS = registry
    raw = {id(ref_fp._div_rem): "div_rem", id(ref_fp._sqrt_resid): "sqrt_resid"}
    by_core = {id(c): n for n, c in ref_core_of.items()}

    def _factory(core):
        if id(core) in raw:
            return ours.raw_loop(raw[id(core)])
        if id(core) in by_core:
            return ours.KERNELS[by_core[id(core)]].loop
        raise NotImplementedError("no device loop for core %r" % (core,))

    shim._loop22 = shim._loop21 = shim._loop11 = shim._loop1u = _factory
    shim.__all__ = list(ours.__all__)
    sys.modules["twofold.kernels"] = shim
    twofold.kernels = shim
    twofold.TwofoldArray = ours.TwofoldArray
    twofold.CoupledArray = ours.CoupledArray
    twofold.empty_twofold = ours.empty_twofold
    del ref_arith
    return shim


SHIM = install()


def pytest_report_header(config):
    import twofold

    from paper_1401_6235_b200 import _lib

    return ["refsuite shim: twofold.kernels -> paper_1401_6235_b200.kernels (%s); reference "
            "package %s; gmpy2 %s" % (_lib.LIB_PATH, twofold.__file__,
                                      "stub (fractions.Fraction)"
                                      if getattr(sys.modules["gmpy2"], "__stub__", False)
                                      else "real")]
