"""Fold `ncu --set full` captures of the bench shapes (tools/gpu_ncu_shapes.sh)
into profiles/ncu_traffic.json, keyed "op|dtype|n" (bench.ncu_traffic), and a
per-kernel summary next to it.

    python tools/ncu_traffic_update.py gpurun_out/ns_config2.ncu-rep ... --tag r2

A `.summary.json` (tools/ncu_summary.py --json, written on the GPU box when the reports
are too large to bring back) is accepted in place of a report.
"""
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summarise  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
OPS = ["vtadd2", "vtsub2", "vtmul2", "vtdiv2", "vtadd1", "vtsub1", "vtmul1", "vtdiv1", "vtadd",
       "vtsub", "vtmul", "vtdiv", "vtsqrt1", "vtsqrt", "vpadd2", "vpsub2", "vpmul2", "vpdiv2",
       "vpadd1", "vpsub1", "vpmul1", "vpdiv1", "div_rem", "sqrt_resid"]
N = {"config1": 1 << 20, "config2": 1 << 28, "config3": 1 << 30, "config4": 1 << 30,
     "config5": 1 << 26}
ROPS = {"0": "vtsum", "1": "vtsum2", "2": "vtdot"}


def op_of(kernel):
    m = re.search(r"ew_kernel<(double|float), (\d+), 32>", kernel) or \
        re.search(r"ew_(?:bulk|step|step16)_kernel<(double|float), (\d+)>", kernel)
    if m:
        return OPS[int(m.group(2))], "f64" if m.group(1) == "double" else "f32"
    m = re.search(r"reduce_kernel<(double|float), (\d)", kernel)
    if m:
        return ROPS[m.group(2)], "f64" if m.group(1) == "double" else "f32"
    m = re.search(r"horner_kernel<(double|float)", kernel)
    if m:
        return "vthorner", "f64" if m.group(1) == "double" else "f32"
    return None, None


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else "r2"
    args = [a for a in args if a != tag]
    path = ROOT / "profiles" / "ncu_traffic.json"
    try:
        table = json.loads(path.read_text())
    except Exception:
        table = {}
    table = {k: v for k, v in table.items() if "|" in k}  # drop round-1 unkeyed entries
    summary = []
    for rep in args:
        cfg = re.search(r"(config\d)", rep).group(1)
        rows = json.loads(Path(rep).read_text()) if rep.endswith(".json") else summarise(rep)
        for d in rows:
            op, dt = op_of(d["kernel"])
            if op is None:
                continue
            key = "%s|%s|%d" % (op, dt, N[cfg])
            rec = {"dram_bytes": d["dram_traffic"], "dram_read": d["dram_read"],
                   "dram_write": d["dram_write"], "time_ms": d["time"] * 1e3,
                   "dram_pct_peak": d.get("dram_pct_peak"), "regs": d.get("regs"),
                   "warps_active_pct": d.get("warps_active_pct"),
                   "fp64_pipe_pct": d.get("fp64_pipe_pct"), "fp64_inst": d.get("fp64_inst"),
                   "source": "%s (%s, ncu --set full --clock-control none)"
                             % (Path(rep).name.replace(".summary.json", ".ncu-rep"), tag)}
            table[key] = rec
            summary.append(dict(key=key, kernel=d["kernel"][:90], **rec))
    path.write_text(json.dumps(dict(sorted(table.items())), indent=1) + "\n")
    (ROOT / "profiles" / ("%s_ncu_shapes.json" % tag)).write_text(json.dumps(summary, indent=1) + "\n")
    for s in summary:
        print("%-28s %8.3f ms  %7.2f GB  dram%%peak %5.1f  regs %s" % (
            s["key"], s["time_ms"], s["dram_bytes"] / 1e9, s["dram_pct_peak"] or 0, s["regs"]))


if __name__ == "__main__":
    main()
