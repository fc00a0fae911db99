"""CPU checks of bench.py's contract pieces that need no GPU: the reference arm
prints one JSON line with the required keys (small sample)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


import pytest


@pytest.mark.parametrize("workload", ["config2", "config4", "config5"])
def test_reference_arm_json_line(workload):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--workload", workload, "--steps", "2", "--warmup", "1",
                        "--cpu-sample", "65536"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
    assert ("configs[%d]" % {"config2": 1, "config4": 3, "config5": 4}[workload]) in d["config"]["workload"]


def test_reference_arm_non_zero_ranks_exit_quietly():
    env = {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}
    import os

    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       timeout=120, cwd=ROOT, env=e)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_exact_check_of_a_generated_dot(oracle):
    # the config-4 full-size check on a small instance: the calibrated generator
    # hits the requested condition and the canonical-order twofold is in bound
    import numpy as np

    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1401_6235_b200 import _lib

    n = 1 << 15
    x, y = np.empty(n), np.empty(n)
    assert _lib.lib().tf_gen_dot_host(n, 1e16, 4242, x.ctypes.data, y.ctypes.data) == 0
    zd = oracle.reduce("dot", x, y, geometry=(2, 256, 128))
    zs = oracle.reduce("sum", x, geometry=(2, 256, 128))
    c = bench.exact_check(x, y, [float(zd[0]), float(zd[1])], [float(zs[0]), float(zs[1])], 2)
    assert c["vtdot"]["bound_ok"] and c["vtsum"]["bound_ok"]
    assert 0.5e16 < c["vtdot"]["cond"] < 2e16
    assert c["vtdot"]["z0_plus_z1_rel_err"] < 1e-10 < c["vtdot"]["z0_rel_err"]


REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
            "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks")


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["config2", "config4", "config5"])
def test_our_arm_json_line_contract(workload):
    # the driver's contract on our arm, at a small size: one JSON line with every
    # required key, the roofline / cpu_baseline / e2e / clocks objects filled, and
    # the full-size checks of the timed outputs passing
    elems = {"config2": 1 << 22, "config4": 1 << 23, "config5": 1 << 22}[workload]
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--workload", workload,
                        "--elems", str(elems), "--steps", "3", "--warmup", "3",
                        "--cpu-sample", str(1 << 20), "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["scaling"] == "weak" and d["higher_is_better"] is True
    assert "workload" in d["config"]
    rl = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rl, k
    assert rl["achieved"] > 0 and rl["peak"] > 0
    cb = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in cb, k
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k
    if workload == "config2":
        chk = d["device_batch"]["check"]
        assert all(v for op, c in chk.items() if op != "how" for v in c.values()), chk
    elif workload == "config4":
        assert d["device_batch"]["same_bits_as_separate_reductions"] is True
        assert d["cpu_baseline"]["check"]["vtdot"]["bound_ok"] is True
    else:
        assert d["check"]["flag_rate"] > 0.99
