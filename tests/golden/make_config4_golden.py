"""Golden bits for BASELINE config 4 (f64 vtdot + vtsum, n = 2^30, cond 1e16).

    python tests/golden/make_config4_golden.py   # ~24 GiB of host RAM, a few minutes

Generates the config-4 planes on the HOST (tf_gen_ill_host: the blocked
Ogita-Rump-Oishi-style generator, csrc/gen_ill.cu; bit-identical to the device
generator, tests/test_gpu_gen_ill.py) and reduces every power-of-two prefix
from 2^16 to 2^30 with the CPU oracle in the canonical order
(oracle/twofold_oracle.c — the checker, pinned to the reference's own numba
cores by tests/test_oracle_golden.py).  The exact integer-limb accumulator
gives the exact dot / sum, sum|terms| and the achieved condition numbers:

    cond(dot)  = 2 sum|x_i y_i| / |sum x_i y_i|   (Ogita-Rump-Oishi's definition)
    cond1(dot) =   sum|x_i y_i| / |sum x_i y_i|
    cond(sum)  =   sum|p_i| / |sum p_i|

and |(z0 + z1) - exact| / (4u sum|terms|) for the canonical-order results.
A prefix of whole generator blocks is itself a config-4 problem (every block
is calibrated), which is what the multi-rank bench shards and the dry runs use.
Output: tests/golden/config4.json (z0/z1 as float.hex, exact figures as floats).
"""

from __future__ import annotations

import json
import os
import sys
import time
from fractions import Fraction
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as o  # noqa: E402
from paper_1401_6235_b200 import workloads as W  # noqa: E402


def main(top=30):
    n = 1 << top
    t0 = time.time()
    x = np.empty(n)
    y = np.empty(n)
    p = np.empty(n)
    W.gen_ill(W.GEN_DOT, x, y)
    W.gen_ill(W.GEN_SUM, p)
    print("generated 2^%d in %.1f s" % (top, time.time() - t0), flush=True)
    u4 = 4 * Fraction(1, 2**53)
    out = {"generator": {"cond": W.C4_COND, "seed": W.C4_SEED, "emin": W.C4_EMIN,
                         "emax": W.C4_EMAX, "block": W.GEN_BLOCK,
                         "how": "tf_gen_ill_host (csrc/gen_ill.cu), prefixes of the 2^%d problem"
                                % top},
           "geometry": [2, 256, 128], "prefixes": {}}
    for k in range(16, top + 1):
        m = 1 << k
        rec = {}
        for name, rop, planes in (("vtdot", "dot", (x[:m], y[:m])), ("vtsum", "sum", (p[:m],))):
            z0, z1 = o.reduce(rop, *planes, geometry=(2, 256, 128))
            s, t = o.exact(rop, *planes)
            err = abs(Fraction(float(z0)) + Fraction(float(z1)) - s)
            rec[name] = {"z0": float(z0).hex(), "z1": float(z1).hex(),
                         "exact": float(s), "sum_abs_terms": float(t),
                         "cond": float((2 if rop == "dot" else 1) * t / abs(s)),
                         "cond1": float(t / abs(s)),
                         "err_over_4u_bound": float(err / (u4 * t)),
                         "z0_rel_err": float(abs(Fraction(float(z0)) - s) / abs(s)),
                         "z0_plus_z1_rel_err": float(err / abs(s))}
        out["prefixes"][str(m)] = rec
        print(k, {nm: (r["cond"], r["err_over_4u_bound"]) for nm, r in rec.items()},
              "%.1f s" % (time.time() - t0), flush=True)
    (ROOT / "tests" / "golden" / "config4.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main(int(os.environ.get("C4_TOP", "30")))
