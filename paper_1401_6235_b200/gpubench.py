"""GPU backend for the reference's throughput harness (``twofold bench``).

Mirrors /root/reference/pkg/src/twofold/bench.py: the same plan cells
(``make_plan``, bench.py:184-199), the same dotted baselines vadd/vmul/vdiv/
vsqrt/vmem (bench.py:56-87), the same seeded inputs (crc32 of "op:fmt:n",
magnitudes in [1,2) with random signs, tails 2^-54 / 2^-25 below; bench.py:131-162),
the same best-of-N measurement that grows the repeat count until one
measurement spans >= 10 ms (bench.py:165-181), and the same CSV layout
(bench.py:270-279) with GPU columns appended.

The reference times a compiled repeat loop so no interpreter sits in the timed
region; here the repeat loop is a CUDA graph of ``iters`` kernel launches,
replayed and timed with CUDA events on the capturing stream.

    python -m paper_1401_6235_b200.gpubench --ops vtadd2,vtdiv2 --sizes large,hbm \
        --format f64 --csv out.csv

``ratio_vs_dotted`` = dotted Mops / twofold Mops (bench.py:264-266).  Extra
columns: gpus, gbps (algorithmic bytes / time), roofline_frac (gbps / measured
HBM peak), bytes_per_elem, ops_per_elem (floating-point operations of the core).
"""

from __future__ import annotations

import argparse
import csv
import json
import re
import zlib
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import numpy as np

from . import _lib
from .kernels import KERNELS

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

# reference size classes (bench.py:32) plus an HBM-bound class
SIZES = {"small": 100, "medium": 10_000, "large": 1_000_000, "hbm": 1 << 27}
_FORMATS = {"f32": np.float32, "f64": np.float64}
_BASELINE_FOR = {"add": "vadd", "sub": "vadd", "mul": "vmul", "div": "vdiv", "sqrt": "vsqrt"}
_DOTTED_ID = {"vadd": 0, "vmul": 1, "vdiv": 2, "vsqrt": 3, "vmem": 4}

# floating-point operations per element of each core (div/sqrt count as one)
OPS_PER_ELEM = {
    "vtadd2": 8, "vtsub2": 8, "vtmul2": 8, "vtdiv2": 6, "vtadd1": 7, "vtsub1": 7,
    "vtmul1": 4, "vtdiv1": 4, "vtadd": 6, "vtsub": 6, "vtmul": 2, "vtdiv": 3,
    "vtsqrt1": 20, "vtsqrt": 4, "vpadd2": 11, "vpsub2": 11, "vpmul2": 12, "vpdiv2": 8,
    "vpadd1": 10, "vpsub1": 10, "vpmul1": 10, "vpdiv1": 7,
    "vadd": 1, "vmul": 1, "vdiv": 1, "vsqrt": 1, "vmem": 0,
}
_NIN = {"22": 4, "21": 3, "11": 2, "u2": 2, "u1": 1}


@dataclass
class BenchRecord:
    op: str
    shape: str
    format: str
    size_class: str
    elements: int
    mega_ops: float
    ratio_vs_dotted: Optional[float]
    gpus: int = 1
    gbps: float = 0.0
    roofline_frac: float = 0.0
    bytes_per_elem: int = 0
    ops_per_elem: int = 0


def _selection(kind, given, known, hint=""):
    """The reference harness's selection rule (bench.py:184-199): None means every
    known entry; an unknown name is a ValueError naming it."""
    picked = list(known) if given is None else list(given)
    bad = [x for x in picked if x not in known]
    if bad:
        raise ValueError("unknown %s %r%s" % (kind, bad[0], hint))
    return picked


def make_plan(ops=None, formats=None, sizes=None):
    """Plan cells (op, arity, format, size class), format-major then size then op —
    the reference's cell order (bench.py:184-199)."""
    ops = _selection("op", ops, KERNELS)
    formats = _selection("format", formats, _FORMATS, " (use f32/f64)")
    sizes = _selection("size class", sizes, SIZES)
    cells = []
    for fmt in formats:
        for size in sizes:
            cells.extend((op, KERNELS[op].arity, fmt, size) for op in ops)
    return cells


def _cell_seed(op, fmt, n):
    # the reference's per-cell seed (bench.py:144-145): crc32 of "op:fmt:n"
    return zlib.crc32(f"{op}:{fmt}:{n}".encode())


def _value_and_tail(gen, n, dtype, signed=True):
    """Magnitudes in [1, 2) (random sign unless `signed` is False) and a tail
    2^-54 (f64) / 2^-25 (f32) below each, drawn in the reference's order
    (bench.py:148-153) so the planes match its inputs value for value."""
    v = gen.uniform(1.0, 2.0, n)
    if signed:
        v *= gen.choice((-1.0, 1.0), n)
    v = v.astype(dtype)
    tail_scale = dtype(2.0 ** -54) if dtype is np.float64 else dtype(2.0 ** -25)
    return v, (v * tail_scale).astype(dtype)


# planes of x and of y each arity takes: (x value[, x error]), (y value[, y error])
_TAKE = {"22": (2, 2), "21": (2, 1), "11": (1, 1), "u2": (2, 0), "u1": (1, 0)}


def inputs(op, fmt, n):
    """Seeded host planes for one cell, the same values the reference harness
    feeds its loops (bench.py:156-162)."""
    spec = KERNELS[op]
    dtype = _FORMATS[fmt]
    gen = np.random.default_rng(_cell_seed(op, fmt, n))
    nx, ny = _TAKE[spec.arity]
    planes = list(_value_and_tail(gen, n, dtype, signed=spec.baseline != "sqrt"))[:nx]
    if ny:
        planes += list(_value_and_tail(gen, n, dtype))[:ny]
    return tuple(planes)


def _measure(launch, repetitions, min_s=0.010, max_iters=1 << 14):
    """CUDA-graph repeat loop: grow iters until one replay lasts >= min_s,
    then best of `repetitions` replays; returns (iters, seconds)."""
    stream = torch.cuda.Stream()
    iters = 8
    while True:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            launch()  # warm (occupancy query, self-test) outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(iters):
                launch()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        with torch.cuda.stream(stream):
            g.replay()
        b.record(stream)
        b.synchronize()
        dt = a.elapsed_time(b) * 1e-3
        if dt >= min_s or iters >= max_iters:
            break
        iters *= 2
    best = dt
    for _ in range(repetitions - 1):
        a.record(stream)
        with torch.cuda.stream(stream):
            g.replay()
        b.record(stream)
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return iters, best


def _peak_gbs():
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


def _dotted_launcher(name, dt, n, x, y, r):
    base = _DOTTED_ID[name]
    L = _lib.lib()

    def launch():
        s = torch.cuda.current_stream().cuda_stream
        _lib.check(L.tf_dotted(base, dt, n, x.data_ptr(), y.data_ptr() if y is not None else None,
                               r.data_ptr(), s), name)
    return launch


def _il_args(spec, planes):
    from . import interleaved as IL
    from .kernels import TwofoldArray

    ar = spec.arity
    if ar == "22":
        return (IL.from_split(TwofoldArray(planes[0], planes[1])),
                IL.from_split(TwofoldArray(planes[2], planes[3])))
    if ar == "21":
        return (IL.from_split(TwofoldArray(planes[0], planes[1])), planes[2])
    if ar == "u2":
        return (IL.from_split(TwofoldArray(planes[0], planes[1])), None)
    if ar == "11":
        return (planes[0], planes[1])
    return (planes[0], None)


def run_bench(plan=None, repetitions=5, device=0, layout="split"):
    """Measure every plan cell plus the dotted baselines (bench.py:226-267).
    layout="interleaved" times the (n, 2) pair-array kernels instead."""
    if repetitions < 3:
        raise ValueError("repetitions must be >= 3 to filter noise")
    if plan is None:
        plan = make_plan()
    torch.cuda.set_device(device)
    _lib.ensure_device(device)
    peak = _peak_gbs()
    grouped = {}
    for cell in plan:
        op, shape, fmt, size = cell
        spec = KERNELS.get(op)
        if spec is None:
            raise ValueError("unknown op %r" % op)
        if shape != spec.arity:
            raise ValueError("op %s has shape %s, plan says %s" % (op, spec.arity, shape))
        grouped.setdefault((fmt, size), []).append((op, spec))
    records, dotted = [], {}
    for (fmt, size), cells in grouped.items():
        n = SIZES[size]
        dtype = _FORMATS[fmt]
        esz = np.dtype(dtype).itemsize
        tdt = torch.float64 if dtype is np.float64 else torch.float32
        dt = _lib.TF_F64 if dtype is np.float64 else _lib.TF_F32
        for name in ("vadd", "vmul", "vdiv", "vsqrt", "vmem"):
            gen = np.random.default_rng(_cell_seed(name, fmt, n))
            x = torch.from_numpy(_value_and_tail(gen, n, dtype, name != "vsqrt")[0]).cuda()
            unary = name in ("vsqrt", "vmem")
            y = None if unary else torch.from_numpy(_value_and_tail(gen, n, dtype)[0]).cuda()
            r = torch.empty(n, dtype=tdt, device="cuda")
            iters, best = _measure(_dotted_launcher(name, dt, n, x, y, r), repetitions)
            mega = n * iters / best / 1e6
            bpe = (2 if unary else 3) * esz
            gbps = bpe * n * iters / best / 1e9
            records.append(BenchRecord(name, "u1" if unary else "11", fmt, size, n, mega,
                                       None if name == "vmem" else 1.0, 1, gbps, gbps / peak,
                                       bpe, OPS_PER_ELEM[name]))
            dotted[(name, fmt, size)] = mega
        for op, spec in cells:
            planes = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in inputs(op, fmt, n)]
            if layout == "interleaved":
                from . import interleaved as IL

                xa, ya = _il_args(spec, planes)
                po = torch.empty((n, 2), dtype=tdt, device="cuda")
                il = IL.KERNELS[op].launch
                iters, best = _measure(lambda: il(xa, ya, po), repetitions)
            else:
                out = [torch.empty(n, dtype=tdt, device="cuda") for _ in range(2)]
                loop = spec.loop
                iters, best = _measure(lambda: loop(*planes, *out), repetitions)
            mega = n * iters / best / 1e6
            bpe = (_NIN[spec.arity] + 2) * esz
            gbps = bpe * n * iters / best / 1e9
            base = dotted[(_BASELINE_FOR[spec.baseline], fmt, size)]
            records.append(BenchRecord(op, spec.arity, fmt, size, n, mega, base / mega, 1, gbps,
                                       gbps / peak, bpe, OPS_PER_ELEM[op]))
    return records


# (column, CSV format, table header, table format); the first seven are the
# reference's stable CSV layout (bench.py:270-279), the rest are GPU columns
_COLUMNS = [
    ("op", "%s", "op", "%-8s"), ("shape", "%s", "shape", "%-5s"),
    ("format", "%s", "fmt", "%-4s"), ("size_class", "%s", "size", "%-6s"),
    ("elements", "%d", "elements", "%10d"), ("mega_ops", "%.3f", "mega_ops", "%12.1f"),
    ("ratio_vs_dotted", "%.4f", "ratio", "%8.2f"), ("gpus", "%d", None, None),
    ("gbps", "%.1f", "GB/s", "%9.1f"), ("roofline_frac", "%.4f", "roof", "%7.3f"),
    ("bytes_per_elem", "%d", None, None), ("ops_per_elem", "%d", None, None),
]
CSV_HEADER = [c[0] for c in _COLUMNS]


def write_csv(records, path):
    """Records as CSV: the reference's columns, then the GPU columns.  A missing
    ratio (vmem has no dotted baseline) is an empty field."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_HEADER)
        for r in records:
            w.writerow(["" if getattr(r, name) is None else fmt % getattr(r, name)
                        for name, fmt, _, _ in _COLUMNS])


def format_table(records) -> str:
    """Fixed-width table of the records, in the order they arrive."""
    cols = [(name, head, fmt) for name, _, head, fmt in _COLUMNS if head]
    width = lambda fmt: int(re.match(r"%-?(\d+)", fmt).group(1))  # noqa: E731
    out = [" ".join(head.ljust(width(fmt)) if fmt.startswith("%-") else head.rjust(width(fmt))
                    for _, head, fmt in cols)]
    for r in records:
        cells = []
        for name, _, fmt in cols:
            v = getattr(r, name)
            cells.append("-".rjust(width(fmt)) if v is None else fmt % v)
        out.append(" ".join(cells))
    return "\n".join(out) + "\n"


def main(argv=None):
    ap = argparse.ArgumentParser(prog="gpubench", description=__doc__.splitlines()[0])
    ap.add_argument("--ops", help="comma-separated kernel names (default: all)")
    ap.add_argument("--sizes", help="comma-separated size classes (default: all)")
    ap.add_argument("--format", dest="formats", help="comma-separated f32,f64 (default: both)")
    ap.add_argument("--csv", help="also write records to this CSV path")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--layout", choices=["split", "interleaved"], default="split")
    a = ap.parse_args(argv)
    sp = lambda t: None if t is None else [s for s in t.split(",") if s]  # noqa: E731
    recs = run_bench(make_plan(sp(a.ops), sp(a.formats), sp(a.sizes)), repetitions=a.reps,
                     layout=a.layout)
    print(format_table(recs), end="")
    if a.csv:
        write_csv(recs, a.csv)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
