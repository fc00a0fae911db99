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
                        "--ref-elems", "65536"],
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
    # the arm is the stronger of the C port and the reference package itself (numba,
    # fork-sharded) where the latter runs; both are recorded
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    if workload == "config2":
        assert d["port"]["value"] > 0
        nb = d.get("numba_reference")
        if nb and "value" in nb:
            assert d["value"] == max(d["port"]["value"], nb["value"])
            assert d["cpu_baseline"]["kind"] == ("reference" if nb["value"] > d["port"]["value"]
                                                 else "port")
    assert "workload" in d["config"]
    assert ("configs[%d]" % {"config2": 1, "config4": 3, "config5": 4}[workload]) in d["config"]["workload"]
    # the reference arm's config object is the one our arm prints for the workload
    import bench

    n = {"config2": 1 << 28, "config4": 1 << 30, "config5": 1 << 26}[workload]
    assert d["config"] == bench.wl_config(workload, n)
    if workload == "config2":  # the default run carries every other BASELINE config
        assert sorted(d["workloads"]) == ["config1", "config3", "config4", "config5"]
        for wl, rec in d["workloads"].items():
            assert rec["value"] > 0 and rec["config"] == bench.wl_config(wl, bench.WL[wl]["n"])


def test_reference_arm_non_zero_ranks_exit_quietly():
    env = {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}
    import os

    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       timeout=120, cwd=ROOT, env=e)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_exact_check_of_a_generated_problem(oracle):
    # the config-4 full-size check on a small instance: the blocked generator
    # hits the requested condition and the canonical-order twofolds are in bound
    import numpy as np

    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1401_6235_b200 import workloads as W

    n = 1 << 17
    x, y, p = np.empty(n), np.empty(n), np.empty(n)
    W.gen_ill(W.GEN_DOT, x, y)
    W.gen_ill(W.GEN_SUM, p)
    zd = oracle.reduce("dot", x, y, geometry=(2, 256, 128))
    zs = oracle.reduce("sum", p, geometry=(2, 256, 128))
    c = bench.exact_check({"vtdot": (x, y), "vtsum": (p,)}, {"vtdot": zd, "vtsum": zs}, 2)
    assert c["vtdot"]["bound_ok"] and c["vtsum"]["bound_ok"]
    assert 0.5e16 < c["vtdot"]["cond"] < 2e16 and 0.5e16 < c["vtsum"]["cond"] < 2e16
    assert c["vtdot"]["cond1"] == pytest.approx(c["vtdot"]["cond"] / 2)
    for k in ("vtdot", "vtsum"):
        assert c[k]["z0_plus_z1_rel_err"] < 1e-14 < c[k]["z0_rel_err"]


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
                        "--cpu-sample", str(1 << 20), "--e2e-steps", "1",
                        "--no-sub-workloads"],
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
        chk = d["check"]
        ops = d["config"]["ops"]
        assert all(v for op in ops for v in chk[op].values()), chk
        assert all(chk["oracle_sample"]["bit_exact_vs_oracle"].values()), chk
        assert chk["batch_equals_per_op_launch"] and all(chk["batch_equals_per_op_launch"].values())
        pg = d["e2e"]["pageable"]
        assert pg["first_step"] > 0 and pg["steady_state"] > 0
    elif workload == "config4":
        chk = d["check"]
        assert all(chk["bit_exact_vs_oracle"].values()), chk
        for k in ("vtdot", "vtsum"):
            assert chk["exact"][k]["bound_ok"] is True
            assert 0.5e16 < chk["exact"][k]["cond"] < 2e16
        assert all(chk["golden_bits_equal"].values()), chk
    else:
        assert d["check"]["flag_rate"] > 0.99
