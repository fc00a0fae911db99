"""The C ABI from a pure-C client (tests/c_abi/abi_smoke.c): compiled with gcc
against include/twofold_b200.h and linked to libtwofold_b200.so only."""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_1401_6235_b200" / "_lib"


def _build(tmp_path):
    cc = shutil.which("gcc") or "/usr/bin/gcc"
    exe = tmp_path / "abi_smoke"
    cmd = [cc, "-O1", "-std=c99", "-I", str(ROOT / "include"), str(ROOT / "tests" / "c_abi" / "abi_smoke.c"),
           "-L", str(LIBDIR), "-ltwofold_b200", "-Wl,-rpath," + str(LIBDIR), "-lm", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_client_validation(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe), "cpu"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_smoke cpu ok" in r.stdout


@pytest.mark.gpu
def test_c_client_known_answers_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_smoke gpu ok" in r.stdout
