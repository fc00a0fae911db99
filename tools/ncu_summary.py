"""Summarise an ncu --set full report: per-kernel time, DRAM bytes, throughput,
occupancy, FP64-pipe use.  Usage: python tools/ncu_summary.py REPORT.ncu-rep [--json]"""
import csv, io, json, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__inst_executed_pipe_fp64.sum", "fp64_inst"),
    ("smsp__inst_executed.sum", "inst"),
    ("lts__t_bytes.sum", "l2_bytes"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ms": 1e-3}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, short in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    pass
                d[short] = v
        if "dram_read" in d and "dram_write" in d:
            d["dram_traffic"] = d["dram_read"] + d["dram_write"]
        out.append(d)
    return out


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    if "--json" in sys.argv:
        print(json.dumps(res, indent=1))
    else:
        for d in res:
            print(d["kernel"][:70])
            print("   time %.3f ms  dram %.3f GB (r %.3f w %.3f)  %.1f GB/s  dram%%peak %.1f  regs %s grid %s  warps %.1f%%  fp64pipe %.1f%%" % (
                d["time"] * 1e3, d["dram_traffic"] / 1e9, d["dram_read"] / 1e9, d["dram_write"] / 1e9,
                d["dram_traffic"] / d["time"] / 1e9, d["dram_pct_peak"], d.get("regs"), d.get("grid"),
                d.get("warps_active_pct", 0), d.get("fp64_pipe_pct", 0)))
