"""The GPU bench harness keeps the reference harness's plan/CSV contract
(test_bench.py:1-145 in the reference): plan expansion and validation, seeded
inputs, CSV header and the empty vmem ratio; GPU columns appended."""

import csv

import numpy as np
import pytest

from paper_1401_6235_b200 import gpubench as gb


def test_make_plan_expands_and_validates():
    plan = gb.make_plan(["vtadd2", "vtsqrt"], ["f64"], ["small", "large"])
    assert plan == [("vtadd2", "22", "f64", "small"), ("vtsqrt", "u1", "f64", "small"),
                    ("vtadd2", "22", "f64", "large"), ("vtsqrt", "u1", "f64", "large")]
    assert len(gb.make_plan()) == 22 * 2 * len(gb.SIZES)
    for bad in (dict(ops=["nope"]), dict(formats=["f16"]), dict(sizes=["huge"])):
        with pytest.raises(ValueError):
            gb.make_plan(**bad)


def test_inputs_are_seeded_and_well_scaled():
    a = gb.inputs("vtadd2", "f64", 100)
    b = gb.inputs("vtadd2", "f64", 100)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert len(a) == 4 and np.all(np.abs(a[0]) >= 1) and np.all(np.abs(a[0]) < 2)
    s = gb.inputs("vtsqrt", "f32", 50)
    assert len(s) == 1 and s[0].dtype == np.float32 and np.all(s[0] > 0)
    assert np.all(a[1] == a[0] * 2.0**-54)


def _records():
    R = gb.BenchRecord
    return [R("vmem", "u1", "f64", "small", 100, 10.0, None, 1, 1.0, 0.001, 16, 0),
            R("vadd", "11", "f64", "small", 100, 9.0, 1.0, 1, 1.0, 0.001, 24, 1),
            R("vtadd2", "22", "f64", "small", 100, 4.5, 2.0, 1, 1.0, 0.001, 48, 8)]


def test_csv_round_trip(tmp_path):
    p = tmp_path / "b.csv"
    gb.write_csv(_records(), p)
    rows = list(csv.reader(open(p, newline="")))
    assert rows[0][:7] == ["op", "shape", "format", "size_class", "elements", "mega_ops",
                           "ratio_vs_dotted"]
    assert rows[0][7:] == ["gpus", "gbps", "roofline_frac", "bytes_per_elem", "ops_per_elem"]
    by = {r[0]: r for r in rows[1:]}
    assert by["vmem"][6] == "" and float(by["vadd"][6]) == 1.0
    assert int(by["vtadd2"][4]) == 100 and float(by["vtadd2"][5]) > 0


def test_format_table():
    lines = gb.format_table(_records()).splitlines()
    assert lines[0].split()[:7] == ["op", "shape", "fmt", "size", "elements", "mega_ops", "ratio"]
    assert len(lines) == 4 and any("vtadd2" in ln for ln in lines)


def test_ops_per_elem_covers_registry():
    from paper_1401_6235_b200.kernels import KERNELS

    assert set(KERNELS) <= set(gb.OPS_PER_ELEM)


@pytest.mark.gpu
def test_gpu_bench_runs_and_ratios_are_sane(tmp_path):
    recs = gb.run_bench(gb.make_plan(["vtadd2", "vtdiv2", "vtsqrt1"], ["f64"], ["small", "large"]),
                        repetitions=3)
    names = [r.op for r in recs]
    assert names.count("vmem") == 2 and names.count("vtadd2") == 2
    for r in recs:
        assert r.mega_ops > 0
        if r.op.startswith("vt"):
            assert 0 < r.ratio_vs_dotted < 20
    gb.write_csv(recs, tmp_path / "x.csv")
