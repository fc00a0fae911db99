"""Every selectable kernel variant is parity-checked: the A/B switches
(TF_VEC_BYTES=16, TF_EW_SCHED=persistent, TF_EW_LEAN=0 / TF_EW_REPS — the chunked
ew_kernel instead of the lean single-step kernel —, TF_EW_V16=all/0 — the lean 16-byte
kernel for every op / none —, TF_BATCH_V16=1, TF_CONV_LEAN=1/0, TF_EW_BULK=0/all — the register
and TMA-staged elementwise paths for every op —, TF_REDUCE_PATH=bulk, the host pipeline's
slots/chunks and its zero-copy threshold TF_HOST_ZEROCOPY_MB) are read once per
process, so each runs tools/sanitize_smoke.py (all kernel families, odd sizes,
misaligned views, partial tiles, vs the oracle) in its own subprocess."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

VARIANTS = [{}, {"TF_VEC_BYTES": "16"}, {"TF_EW_SCHED": "persistent"},
            {"TF_EW_BULK": "0"}, {"TF_EW_BULK": "all"}, {"TF_EW_BULK": "all", "TF_EW_BULK_REPS": "3"},
            {"TF_EW_LEAN": "0"}, {"TF_EW_REPS": "2"}, {"TF_EW_V16": "all"}, {"TF_EW_V16": "0"},
            {"TF_BATCH_V16": "1"}, {"TF_CONV_LEAN": "1"}, {"TF_CONV_LEAN": "0"}, {"TF_BATCH_LEAN": "0"}, {"TF_IL_LEAN": "1"},
            {"TF_REDUCE_PATH": "bulk"}, {"TF_HOST_SLOTS": "2", "TF_HOST_CHUNK_MB": "1"},
            {"TF_HOST_ZEROCOPY_MB": "0"}, {"TF_HOST_ZEROCOPY_MB": "4096"}]


@pytest.mark.gpu
@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join("%s=%s" % kv for kv in e.items()) or "default")
def test_variant_parity(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_smoke.py")], env=e,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "mismatches: 0" in r.stdout


@pytest.mark.gpu
def test_fused_32_byte_variant_parity():
    # axpy / submul default to 16-byte vectors; the 32-byte kernels (TF_FUSED_VB=32) must
    # give the same bits: the fused parity tests again in a process with the switch set
    e = dict(os.environ, TF_FUSED_VB="32")
    r = subprocess.run([sys.executable, "-m", "pytest", str(ROOT / "tests" / "test_fused.py"), "-x",
                        "-q", "-m", "gpu", "-p", "no:cacheprovider"], env=e, capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
