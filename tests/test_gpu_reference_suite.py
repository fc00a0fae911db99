"""The reference's OWN hot-path tests, unmodified, against the drop-in on B200.

Runs /root/reference/pkg/tests/test_kernels.py (all of it) and the kernel
criteria 4, 5, 7 and 10 of test_acceptance.py — staged as shipped into
baseline/_ref/twofold_tests by tools/stage_reference.sh, with the reference
package itself in baseline/_ref/twofold — in a subprocess whose
``twofold.kernels`` is this repo's ``paper_1401_6235_b200.kernels``
(tests/refsuite_shim.py).  Every kernel call in those tests passes numpy planes,
so they run end to end through the host pipeline on the device.

Not run, and why: criterion 9 (test_acceptance.py:424-441) times the
reference's CPU bench harness against numba dotted loops on 100-element calls
(the GPU backend of that harness is gpubench.py, its criterion test
tests/test_gpubench.py); criteria 1-3, 6 and 8 and test_arith / test_fp_core /
test_demos / test_cli / test_bench exercise the scalar API, demos and CLI,
which are out of the hot path's scope and untouched by the drop-in.

Skipped when baseline/_ref has not been staged (the GPU box only has what the
repo snapshot carries).
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
SUITE = REF / "twofold_tests"

pytestmark = pytest.mark.gpu

KERNEL_CRITERIA = "criterion_04 or criterion_05 or criterion_07 or criterion_10"


def _run(args, timeout):
    if not (SUITE / "test_kernels.py").exists() or not (REF / "twofold" / "kernels.py").exists():
        pytest.skip("reference not staged into baseline/_ref (tools/stage_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(ROOT / "tests"), str(REF)])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/tf_numba_cache")
    cmd = [sys.executable, "-m", "pytest", "-p", "refsuite_shim", "-c", os.devnull,
           "--rootdir", str(SUITE), "-p", "no:cacheprovider"] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=str(SUITE),
                       env=env)
    tail = (r.stdout + r.stderr)[-4000:]
    print(tail)
    return r, tail


def _passed(tail):
    m = re.search(r"(\d+) passed", tail)
    return int(m.group(1)) if m else 0


def test_reference_test_kernels_unmodified():
    r, tail = _run([str(SUITE / "test_kernels.py")], 1200)
    assert r.returncode == 0, tail
    assert "failed" not in tail and _passed(tail) == 61, tail
    assert "refsuite shim" in r.stdout


def test_reference_acceptance_kernel_criteria_unmodified():
    r, tail = _run([str(SUITE / "test_acceptance.py"), "-k", KERNEL_CRITERIA], 2400)
    assert r.returncode == 0, tail
    assert "failed" not in tail and _passed(tail) == 8, tail
