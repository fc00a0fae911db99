"""Seeded BASELINE-distributed inputs for configs 1-3 (numpy only).

Shared by tests/golden/make_golden.py (which runs the reference on them and
records output digests) and tests/test_config_hashes.py (which re-creates
them on any box and checks the oracle / device outputs against the digests).
"""

import numpy as np


def cfg_inputs(config, name, n, seed):
    rng = np.random.default_rng(seed)
    if config == "config1":
        x0 = rng.uniform(-1, 1, n)
        y0 = rng.uniform(-1, 1, n)
        return [x0, x0 * 2.0**-53 * rng.uniform(-1, 1, n), y0, y0 * 2.0**-53 * rng.uniform(-1, 1, n)]
    if config == "config2":
        def head(lo, hi, signed=True):
            v = np.exp2(rng.uniform(lo, hi, n))
            return v * rng.choice([-1.0, 1.0], n) if signed else v

        def tail(h):
            return h * 2.0**-53 * rng.uniform(-1, 1, n)

        if name == "vtsqrt1":
            x0 = head(-20, 20, False)
            return [x0, tail(x0)]
        x0 = head(-20, 20)
        y0 = head(-10, 10, False) if name == "vtdiv2" else head(-20, 20)
        return [x0, tail(x0), y0, tail(y0)]
    f = np.float32
    x0 = rng.uniform(-1, 1, n).astype(f)
    y0 = (rng.uniform(0.5, 2, n) if name == "vtdiv2" else rng.uniform(-1, 1, n)).astype(f)
    t = lambda h: (h * f(2.0**-24) * rng.uniform(-1, 1, n).astype(f)).astype(f)  # noqa: E731
    return [x0, t(x0), y0, t(y0)]
