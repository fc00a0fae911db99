"""Benchmark of the twofold hot path on B200 — driver contract (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload config2|config1|config3|config4|config5]
                    [--scaling weak|strong] [--elems N] [--no-sub-workloads]

The headline (`value`) is BASELINE.json configs[1]: the full fp64 op set
vtadd2, vtsub2, vtmul2, vtdiv2, vtsqrt1 at n = 2^28 elements per GPU (weak
scaling: every rank owns an independent 2^28-element shard of a global array of
N·2^28; --scaling strong splits one 2^28 array instead).  One step = one pass
of the five kernels.  Inputs are seeded synthetic planes with BASELINE's
distributions, generated on the device before timing; each plane is 2 GiB, far
larger than the 126 MB L2, so no flush is needed between steps.

The default run also measures BASELINE's other configs and reports them under
`workloads` (each with its own value, roofline, cpu_baseline, e2e, check and
clocks, a few steps each):
  config1  f64 vtadd2 + vtmul2, n = 2^20 (parity config; L2 flushed between steps)
  config3  f32 vtadd2 + vtmul2 + vtdiv2, n = 2^30
  config4  f64 vtdot(x, y) + vtsum(p), n = 2^30, cond 1e16 (blocked ORO-style
           generator, every rank generating its shard of ONE global problem);
           per-GPU canonical-order reductions + NCCL all-gather + tf_combine;
           full-size check against the CPU oracle and its exact accumulator
  config5  f64 twofold Horner of the expanded (x-1)^20 at 2^26 points
At N > 1 every record also carries the other scaling mode (`other_scaling`):
strong for the weak headline, with config 4's bits asserted equal to N = 1.

Keys beyond the base contract:
  roofline      dominant kernel: algorithmic bytes (or FP64 instructions) per
                launch / its CUDA-event launch time vs MEASURED_PEAKS.json hbm_gbs;
                traffic = ncu DRAM bytes per launch of that kernel at THIS shape
                (profiles/ncu_traffic.json, keyed kernel|dtype|n), else null
  cpu_baseline  the CPU oracle port (oracle/, all host threads) on a bounded
                sample of the same workload, rank 0 at N=1 only
  e2e           the same metric through the public API on HOST planes, H2D and
                D2H inside: the step as ONE host_batch call over pinned planes;
                e2e.per_call = the reference's convention, one call per op;
                e2e.pageable = per-call on plain (pageable) numpy planes, first
                step and steady state (reused planes get page-locked)
  per_op        per-kernel CUDA-event times and GB/s
  device_batch  the step's ops as ONE launch (kernels.batch -> tf_elementwise_batch)
  clocks        NVML SM clock + event reasons sampled during the timed region

--impl reference times the reference algorithm's CPU implementation — the oracle
port (the numba reference cannot travel to the GPU box) — on all host threads,
on the same config (full size where host RAM allows, else a stated sample).
"""

from __future__ import annotations

import argparse
import copy
import gc
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "twofold elem-ops/s & achieved HBM GB/s (fp64) at 1/2/4/8 B200 vs CPU oracle"
SUB_WORKLOADS = ("config1", "config3", "config4", "config5")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2",
                    choices=["config1", "config2", "config3", "config4", "config5"])
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: n elements per GPU (global N*n); strong: one global "
                         "problem of n elements split over the N GPUs")
    ap.add_argument("--elems", dest="n", type=int, default=0,
                    help="elements per GPU (weak) or in total (strong); default: the config's")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay each step as a CUDA graph (auto: n <= 2^22, launch-bound)")
    ap.add_argument("--reduce-transport", choices=["nccl", "p2p"], default="nccl",
                    help="config4 cross-GPU combine: NCCL all-gather + tf_combine, or each "
                         "reduction fused with the NVLink peer-memory exchange in one launch "
                         "(tf_xgpu_reduce, csrc/xgpu.cu)")
    ap.add_argument("--l2-flush", choices=["write", "write-read"], default="write-read",
                    help="between timed steps of an L2-sized working set: write a 512 MB "
                         "buffer, then (write-read) read another 512 MB so the flush's own "
                         "dirty lines are written back before, not inside, the next step")
    ap.add_argument("--serial-graph", action="store_true",
                    help="small n: capture the step's ops one after another (shared output "
                         "planes) instead of as parallel graph branches")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pageable", action="store_true", help="skip the pageable-numpy e2e leg")
    ap.add_argument("--no-device-batch", action="store_true",
                    help="skip the one-launch-per-step device batch leg (extra output planes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="config4: skip the full-size oracle check")
    ap.add_argument("--no-other-scaling", action="store_true",
                    help="at N > 1, skip the other scaling mode's sub-record")
    ap.add_argument("--no-sub-workloads", action="store_true",
                    help="the default run: skip the configs 1/3/4/5 sub-records")
    ap.add_argument("--sub-steps", type=int, default=10,
                    help="timed steps of each sub-workload (at most --steps)")
    ap.add_argument("--sub-elems", type=int, default=0,
                    help="elements of each sub-workload (default: the config's; dry runs)")
    ap.add_argument("--cpu-sample", type=int, default=1 << 26,
                    help="elements per op in the CPU baseline sample")
    ap.add_argument("--no-numba-ref", action="store_true",
                    help="reference arm: skip timing the numba reference package itself "
                         "(then the arm is the C port alone)")
    ap.add_argument("--ref-elems", type=int, default=0,
                    help="reference arm: elements per op per step (default: the config's "
                         "full size where host RAM allows, else a bounded sample)")
    return ap.parse_args(argv)


_T0 = time.perf_counter()


def log(msg):
    if os.environ.get("RANK", "0") == "0":
        print("[bench %7.1fs] %s" % (time.perf_counter() - _T0, msg), file=sys.stderr, flush=True)


def env_rank():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# --------------------------------------------------------------------------
# measurement helpers


class ClockSampler:
    """NVML SM clock + clock-event reasons, sampled every 10 ms in a thread."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.stop_ev = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()
            if not self.samples:  # a timed region shorter than one sample period
                try:
                    self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                except Exception:
                    pass

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel, dtype, n):
    """DRAM bytes (read + write) per launch of `kernel` at this dtype and size,
    from one `ncu --set full` capture of that exact shape (profiles/
    ncu_traffic.json, keys "kernel|dtype|n"); None when no capture of this shape
    exists — another shape's bytes are never reported."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(p.read_text())
    except Exception:
        return None
    v = d.get("%s|%s|%d" % (kernel, dtype, n))
    if isinstance(v, dict):
        return v.get("dram_bytes")
    return v


_LINK = {}


def link_probe(nbytes=1 << 30):
    """Measured host<->device link (pinned buffers, GB/s): H2D alone, D2H alone,
    and concurrent H2D+D2H total.  The e2e (host-plane) roofline.  Measured
    once per process."""
    import torch

    if _LINK:
        return _LINK
    h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    h2 = torch.empty_like(h, pin_memory=True)
    d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    d2 = torch.empty_like(d)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = float("inf")
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        return best

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    _LINK.update({"h2d": nbytes / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9,
                  "d2h": nbytes / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e9,
                  "duplex": 2 * nbytes / timed(both) / 1e9})
    del h, h2, d, d2
    return _LINK


def link_roofline(h2d, d2h, dt, steps):
    """Time bound of the host link for this traffic mix: each direction alone,
    and both together against the measured duplex total."""
    link = link_probe()
    hb, db = h2d * steps, d2h * steps
    t_bound = max(hb / (link["h2d"] * 1e9), db / (link["d2h"] * 1e9),
                  (hb + db) / (link["duplex"] * 1e9))
    return {"bound": "pcie", "achieved": (hb + db) / dt / 1e9,
            "peak": (hb + db) / t_bound / 1e9, "unit": "GB/s",
            "frac": t_bound / dt, "link_gbs": dict(link),
            "peak_source": "measured live: pinned H2D, D2H and concurrent copies; "
                           "peak = this step's H2D/D2H mix at the link bound"}


def fp64_nominal(sm_mhz=1965.0):
    """148 SMs x 64 FP64 instructions/clk at the max SM clock (instr/s)."""
    return 148 * 64 * sm_mhz * 1e6


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_true(x, world):
    """Logical AND over ranks."""
    if world == 1:
        return bool(x)
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([1 if x else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def release_memory():
    """Between workloads: drop cached device blocks and pinned host blocks."""
    import torch

    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    try:
        torch._C._host_emptyCache()
    except Exception:
        pass


def _pinned_empty(n, esz):
    import torch

    dt = torch.float64 if esz == 8 else torch.float32
    return torch.empty(n, dtype=dt, pin_memory=True).numpy()


def _pinned_copy(t):
    import torch

    h = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


class L2Flush:
    """Cold-L2 flush between timed launches (outside the timed intervals): a
    512 MB memset (larger than the 126 MB L2); with mode write-read, then a read
    of a second 512 MB buffer, which evicts — writes back — the memset's dirty
    lines, so the timed kernel does not pay for the flush's write-back."""

    def __init__(self, mode):
        import torch

        self.mode = mode
        self.w = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.zeros(64 << 20, dtype=torch.int64, device="cuda") \
            if mode == "write-read" else None

    def __call__(self, k):
        self.w.fill_(k & 0xFF)
        if self.r is not None:
            self.r.max()

    def describe(self):
        return ("512 MB memset + 512 MB read between steps" if self.r is not None
                else "512 MB memset between steps") + " (outside the timed intervals)"


def _best_of(fn, reps=3, warm_s=1.0):
    # warm up for ~1 s (thread pool, page faults, and the host CPUs' clocks: on
    # the GPU boxes a cold first second of OpenMP work ran ~1.7x slower,
    # profiles/r2_cpu_probe.json)
    t0 = time.perf_counter()
    fn()
    while time.perf_counter() - t0 < warm_s:
        fn()
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best


# --------------------------------------------------------------------------
# workload descriptions (shared by both arms: identical `config` objects)

WL = {
    "config1": dict(names=["vtadd2", "vtmul2"], dtype=np.float64, n=1 << 20,
                    desc="BASELINE configs[0]: f64 vtadd2+vtmul2, n=2^20 (parity config, L2-resident)"),
    "config2": dict(names=["vtadd2", "vtsub2", "vtmul2", "vtdiv2", "vtsqrt1"], dtype=np.float64,
                    n=1 << 28,
                    desc="BASELINE configs[1]: f64 vtadd2/vtsub2/vtmul2/vtdiv2/vtsqrt1, n=2^28 per GPU"),
    "config3": dict(names=["vtadd2", "vtmul2", "vtdiv2"], dtype=np.float32, n=1 << 30,
                    desc="BASELINE configs[2]: f32 vtadd2/vtmul2/vtdiv2, n=2^30 per GPU"),
    "config4": dict(names=["vtdot", "vtsum"], dtype=np.float64, n=1 << 30,
                    desc="BASELINE configs[3]: f64 vtdot(x, y) + vtsum(p), n=2^30 per GPU, "
                         "cond 1e16 (blocked ORO-style generator, exponents in [-50, 50])"),
    "config5": dict(names=["vthorner"], dtype=np.float64, n=1 << 26,
                    desc="BASELINE configs[4]: twofold Horner (x-1)^20, n=2^26 per GPU"),
}


def wl_config(name, n, scaling="weak"):
    """The `config` object of a line — identical in both arms for one workload."""
    wl = WL[name]
    return {"workload": wl["desc"], ("n_per_gpu" if scaling == "weak" else "n_total"): n,
            "ops": wl["names"]}


def _par_gen(n, fn, seed, dtype=np.float64, like=None):
    """A plane of n values, fn(rng, m[, like_chunk]) per chunk, generated on all
    host threads (numpy's generators release the GIL), one seeded stream per chunk."""
    from concurrent.futures import ThreadPoolExecutor

    nt = max(1, min(os.cpu_count() or 1, 64))
    nch = max(1, min(4 * nt, n // (1 << 16)))
    bounds = [n * i // nch for i in range(nch + 1)]
    seqs = np.random.SeedSequence(seed).spawn(nch)
    out = np.empty(n, dtype)

    def work(i):
        rng = np.random.default_rng(seqs[i])
        lo, hi = bounds[i], bounds[i + 1]
        v = fn(rng, hi - lo) if like is None else fn(rng, hi - lo, like[lo:hi])
        out[lo:hi] = v

    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(work, range(nch)))
    return out


def ref_planes(workload, n, seed=7):
    """Host input planes with the device fill's distributions (BASELINE.json),
    shared between ops the way the device PlaneSet shares them:
    {op: [planes]}.  For the CPU reference arm."""
    def logu(lo, hi, signed):
        def f(rng, m):
            v = np.exp2(rng.uniform(lo, hi, m))
            return v * rng.choice([-1.0, 1.0], m) if signed else v
        return f

    def unif(lo, hi, dt=np.float64):
        return lambda rng, m: rng.uniform(lo, hi, m).astype(dt)

    def tail(p, dt=np.float64):
        return lambda rng, m, h: (h * dt(2.0**p) * rng.uniform(-1, 1, m).astype(dt)).astype(dt)

    if workload == "config2":
        X0 = _par_gen(n, logu(-20, 20, True), seed)
        Y0 = _par_gen(n, logu(-20, 20, True), seed + 1)
        D0 = _par_gen(n, logu(-10, 10, False), seed + 2)
        S0 = _par_gen(n, logu(-20, 20, False), seed + 3)
        X1, Y1, D1, S1 = (_par_gen(n, tail(-53), seed + 10 + k, like=h)
                          for k, h in enumerate((X0, Y0, D0, S0)))
        xy = [X0, X1, Y0, Y1]
        return {"vtadd2": xy, "vtsub2": xy, "vtmul2": xy, "vtdiv2": [X0, X1, D0, D1],
                "vtsqrt1": [S0, S1]}
    if workload == "config3":
        f = np.float32
        X0 = _par_gen(n, unif(-1, 1, f), seed, f)
        Y0 = _par_gen(n, unif(-1, 1, f), seed + 1, f)
        D0 = _par_gen(n, unif(0.5, 2, f), seed + 2, f)
        X1, Y1, D1 = (_par_gen(n, tail(-24, f), seed + 10 + k, f, like=h)
                      for k, h in enumerate((X0, Y0, D0)))
        xy = [X0, X1, Y0, Y1]
        return {"vtadd2": xy, "vtmul2": xy, "vtdiv2": [X0, X1, D0, D1]}
    if workload == "config1":
        X0 = _par_gen(n, unif(-1, 1), seed)
        Y0 = _par_gen(n, unif(-1, 1), seed + 1)
        X1, Y1 = (_par_gen(n, tail(-53), seed + 10 + k, like=h) for k, h in enumerate((X0, Y0)))
        xy = [X0, X1, Y0, Y1]
        return {"vtadd2": xy, "vtmul2": xy}
    raise ValueError(workload)


REF_PLANES = {"config1": 4, "config2": 8, "config3": 6}


def host_ram_available():
    try:
        import psutil

        return psutil.virtual_memory().available
    except Exception:  # pragma: no cover
        return 16 << 30


# --------------------------------------------------------------------------
# elementwise (configs 1-3)


class Op:
    def __init__(self, name, launch, nbytes, units, planes):
        self.name, self.launch, self.nbytes, self.units, self.planes = \
            name, launch, nbytes, units, planes
        self.host_args = None


def _host_call_args(K, arity, hp, out):
    T = K.TwofoldArray
    if arity == "22":
        return (T(hp[0], hp[1]), T(hp[2], hp[3]), out)
    if arity == "21":
        return (T(hp[0], hp[1]), hp[2], out)
    if arity == "11":
        return (hp[0], hp[1], out)
    if arity == "u2":
        return (T(hp[0], hp[1]), out)
    return (hp[0], out)


def elementwise_ops(wlname, n, offset, dev, separate_outputs=False):
    """Device planes (workloads.PlaneSet, BASELINE distributions) + raw launchers.
    The ops share one output pair (they run one after another) unless
    separate_outputs: then each op writes its own planes (independent ops)."""
    import torch

    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import workloads as WLs

    wl = WL[wlname]
    tdt = torch.float64 if wl["dtype"] == np.float64 else torch.float32
    esz = 8 if wl["dtype"] == np.float64 else 4
    ps = WLs.PlaneSet(wlname, n, tdt, dev, offset=offset)
    out = K.empty_twofold(n, tdt, device=dev)
    ops = []
    for name in wl["names"]:
        planes = ps.planes(name)
        if separate_outputs and ops:
            out = K.empty_twofold(n, tdt, device=dev)
        raw = K.KERNELS[name].loop
        args = list(planes) + [out.value, out.error]
        ops.append(Op(name, (lambda raw=raw, args=args: raw(*args)), (len(planes) + 2) * esz * n,
                      n, planes))
        ops[-1].out = out
    return ops, ps, out


def time_steps(args, ops, ws_bytes, world, local, n):
    """Time K steps of `ops` (one launch each) on the current stream: CUDA events
    per launch and per step; a CUDA graph per step for small (launch-bound) n; an
    L2 flush between steps when the working set fits L2.  Returns the timing
    record; elapsed_ms is the max over ranks."""
    import torch

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for op in ops:
            op.launch()
    torch.cuda.synchronize()
    K = args.steps
    use_graph = args.graph == "on" or (args.graph == "auto" and n <= (1 << 22))
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in ops] for _ in range(K)]
    per_op = {}
    branches = False
    flush = ws_bytes < (384 << 20)
    scrub = L2Flush(args.l2_flush) if flush else None
    if use_graph:
        # small, launch-bound steps: one CUDA graph per step, replayed K times
        # (per-op times come from an eager pass with events around each launch)
        for s in range(K):
            for j, op in enumerate(ops):
                if scrub is not None:
                    scrub(j)  # cold L2 for every timed launch
                ev[s][j][0].record(stream)
                op.launch()
                ev[s][j][1].record(stream)
        torch.cuda.synchronize()
        for j, op in enumerate(ops):
            ts = [ev[s][j][0].elapsed_time(ev[s][j][1]) for s in range(K)]
            per_op[op.name] = {"ms": sum(ts) / K, "eager": True}
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        branches = len(ops) > 1 and len({id(op.out) for op in ops}) == len(ops)
        with torch.cuda.graph(g, stream=cap):
            if branches:
                # independent ops (own output planes): parallel graph branches, so
                # one op's ramp and tail overlap the other's
                fork = torch.cuda.Event()
                fork.record(cap)
                joins = []
                for op in ops[1:]:
                    st = torch.cuda.Stream()
                    st.wait_event(fork)
                    with torch.cuda.stream(st):
                        op.launch()
                    j = torch.cuda.Event()
                    j.record(st)
                    joins.append(j)
                ops[0].launch()
                for j in joins:
                    cap.wait_event(j)
            else:
                for op in ops:
                    op.launch()
        g.replay()
        torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K)]
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record(stream)
        for s in range(K):
            if flush:
                scrub(s)
            step_ev[s][0].record(stream)
            if use_graph:
                g.replay()
            else:
                for j, op in enumerate(ops):
                    ev[s][j][0].record(stream)
                    op.launch()
                    ev[s][j][1].record(stream)
            step_ev[s][1].record(stream)
        end.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    if flush:  # the timed region is the sum of the step intervals
        elapsed_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in step_ev), world)
    else:
        elapsed_ms = max_over_ranks(start.elapsed_time(end), world)
    for j, op in enumerate(ops):
        if use_graph:
            avg = per_op[op.name]["ms"]
            share = avg * K / elapsed_ms
        else:
            ts = [ev[s][j][0].elapsed_time(ev[s][j][1]) for s in range(K)]
            avg = sum(ts) / K
            share = sum(ts) / elapsed_ms
        per_op[op.name] = {"ms": avg, "gbs": op.nbytes / (avg * 1e-3) / 1e9,
                           "bytes": op.nbytes, "share": share}
    return {"elapsed_ms": elapsed_ms, "per_op": per_op, "use_graph": use_graph,
            "graph_branches": bool(use_graph and branches),
            "flush": scrub.describe() if flush else None, "clocks": clk.summary(),
            "launches": K * len(ops)}


def ieee_check(ops, outs):
    """Full-size properties of the timed step's own outputs, on the device with
    plain torch ops (one IEEE-RN kernel per op, so no contraction): z0 is bitwise
    the standard IEEE result of the heads for every op (north star); for the
    add/sub ops z1 is bitwise the TwoSum/TwoDiff error plus the tails."""
    import torch

    res = {}
    with torch.no_grad():
        for op, o in zip(ops, outs):
            P = op.planes
            x0 = P[0]
            y0 = P[2] if len(P) == 4 else None
            ieee = {"vtadd2": lambda: x0 + y0, "vtsub2": lambda: x0 - y0,
                    "vtmul2": lambda: x0 * y0, "vtdiv2": lambda: x0 / y0,
                    "vtsqrt1": lambda: torch.sqrt(x0)}.get(op.name)
            if ieee is None:
                continue
            r = {"z0_is_ieee": bool(torch.equal(o.value, ieee()))}
            if op.name in ("vtadd2", "vtsub2"):
                x1, y1 = P[1], P[3]
                if op.name == "vtadd2":
                    s_ = x0 + y0
                    bv = s_ - x0
                    av = s_ - bv
                    e = (x0 - av) + (y0 - bv)
                    z1 = (x1 + y1) + e
                else:
                    s_ = x0 - y0
                    bv = x0 - s_
                    av = s_ + bv
                    e = (x0 - av) + (bv - y0)
                    z1 = (x1 - y1) + e
                r["z1_is_twosum_identity"] = bool(torch.equal(o.error, z1))
                del s_, bv, av, e, z1
            res[op.name] = r
    res["how"] = ("all elements, on the device: torch ops, one IEEE-RN kernel each "
                  "(arith.py:61-64, 74-77 for the error planes)")
    return res


def oracle_sample_check(ops, outs, m=1 << 20):
    """The first m elements of every op's timed outputs against the CPU oracle
    (bit for bit, NaN by position)."""
    from oracle import oracle as o

    res = {}
    for op, out in zip(ops, outs):
        k = min(m, out.value.shape[0])
        ins = [p[:k].cpu().numpy() for p in op.planes]
        w0, w1 = o.elementwise(op.name, *ins)
        g0, g1 = out.value[:k].cpu().numpy(), out.error[:k].cpu().numpy()
        u = np.uint64 if g0.dtype == np.float64 else np.uint32
        ok = all(np.array_equal(np.isnan(a), np.isnan(b)) and
                 np.array_equal(a[~np.isnan(a)].view(u), b[~np.isnan(b)].view(u))
                 for a, b in ((g0, w0), (g1, w1)))
        res[op.name] = ok
    return {"bit_exact_vs_oracle": res, "elements": min(m, outs[0].value.shape[0]),
            "how": "first elements of the timed outputs vs oracle/twofold_oracle.c"}


def device_batch_leg(args, ops, n, esz, peak, world):
    """The step's ops as ONE launch (kernels.batch -> tf_elementwise_batch), each
    op into its own output planes; each distinct input plane is read from HBM
    once.  Reported beside the headline, which stays one launch per op (the
    reference's API).  Returns (record, outputs) — the outputs feed the checks."""
    import torch

    from paper_1401_6235_b200 import kernels as K

    dev = torch.cuda.current_device()
    tdt = torch.float64 if esz == 8 else torch.float32
    outs = [K.empty_twofold(n, tdt, device=dev) for _ in ops]
    calls = [(op.name,) + _host_call_args(K, K.KERNELS[op.name].arity, op.planes, o)
             for op, o in zip(ops, outs)]
    distinct = {p.data_ptr() for op in ops for p in op.planes}
    nbytes = (len(distinct) + 2 * len(ops)) * esz * n
    stream = torch.cuda.current_stream()
    for _ in range(max(1, args.warmup)):
        K.batch(calls)
    flush = (nbytes < (384 << 20))
    scrub = L2Flush(args.l2_flush) if flush else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize()
    for s in range(args.steps):
        if flush:
            scrub(s)
        ev[s][0].record(stream)
        K.batch(calls)
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), world) / args.steps
    gbs = nbytes / (ms * 1e-3) / 1e9
    rec = {"value": world * len(ops) * n / (ms * 1e-3), "unit": "elem-ops/s",
           "ms_per_step": ms, "bytes_per_step": nbytes, "distinct_input_planes": len(distinct),
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                        "frac": gbs / peak},
           "launches_per_step": 1,
           "path": "kernels.batch([%d calls]) -> tf_elementwise_batch: one launch per step, "
                   "each op into its own output planes" % len(ops)}
    return rec, outs


def cpu_baseline_elementwise(ops_names, planes_of, n_sample, reps=3, nthreads=None):
    """Oracle port (plain C, OpenMP, all host threads) on a bounded sample:
    planes_of(name) returns the op's host input planes (the first n_sample
    elements of the bench's own device planes)."""
    from oracle import oracle as o

    t_total = 0.0
    nt = nthreads or os.cpu_count() or 1
    dtype = None
    out = None
    for name in ops_names:
        ins = planes_of(name)
        if out is None:
            dtype = ins[0].dtype
            out = (np.zeros(n_sample, dtype), np.zeros(n_sample, dtype))
        t_total += _best_of(lambda: o.elementwise(name, *ins, nthreads=nt, out=out), reps)
    return len(ops_names) * n_sample / t_total, nt


E2E_MAX = 1 << 27  # host-plane sample per plane (1 GiB f64); 2^26 with several ranks
PAGEABLE_MAX = 1 << 26


def e2e_elementwise(args, ops, ps, n, esz, world, wlname):
    """The step through the public API on host planes (H2D + kernels + D2H in
    the timed region): ONE kernels.host_batch call over pinned planes (headline),
    one kernels.<op>(...) call per op over pinned planes (the reference's calling
    convention), and per-call over plain pageable numpy planes (first step and
    steady state)."""
    from paper_1401_6235_b200 import kernels as K

    ne = min(n, E2E_MAX)
    hcache = {}
    host_planes = []
    for op in ops:
        hp = []
        for key, p in zip(ps.keys[op.name], op.planes):
            if key not in hcache:
                hcache[key] = _pinned_copy(p[:ne])
            hp.append(hcache[key])
        host_planes.append(hp)
    host_out = K.TwofoldArray(_pinned_empty(ne, esz), _pinned_empty(ne, esz))
    calls = [_host_call_args(K, K.KERNELS[op.name].arity, hp, host_out)
             for op, hp in zip(ops, host_planes)]
    funcs = [K.KERNELS[op.name].func for op in ops]

    def per_call_step(cs):
        for f, a in zip(funcs, cs):
            f(*a)

    per_call_step(calls)  # warm the host pipeline (staging buffers, streams)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        per_call_step(calls)
    dt = max_over_ranks(time.perf_counter() - t0, world)
    # the same step as ONE host_batch call: each distinct host plane crosses the
    # link once per chunk; every op writes its own pinned output planes
    bouts = [K.TwofoldArray(_pinned_empty(ne, esz), _pinned_empty(ne, esz)) for _ in ops]
    batch = [(op.name,) + _host_call_args(K, K.KERNELS[op.name].arity, hp, o)
             for op, hp, o in zip(ops, host_planes, bouts)]
    K.host_batch(batch)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        K.host_batch(batch)
    dtb = max_over_ranks(time.perf_counter() - t0, world)
    units = len(ops) * ne
    d2h = 2 * esz * ne * len(ops)
    h2d_call = sum(len(hp) for hp in host_planes) * esz * ne
    h2d_batch = len(hcache) * esz * ne
    rec = {"value": world * units * args.e2e_steps / dtb, "unit": "elem-ops/s",
           "elems_per_op": ne, "h2d_bytes_per_step": h2d_batch, "d2h_bytes_per_step": d2h,
           "roofline": link_roofline(h2d_batch, d2h, dtb, args.e2e_steps),
           "steps": args.e2e_steps,
           "path": "kernels.host_batch([(op, x, y, out) for the %d ops]) on pinned numpy "
                   "planes -> tf_elementwise_host_batch (one chunked H2D / kernels / D2H "
                   "pipeline)" % len(ops),
           "per_call": {"value": world * units * args.e2e_steps / dt,
                        "h2d_bytes_per_step": h2d_call, "d2h_bytes_per_step": d2h,
                        "roofline": link_roofline(h2d_call, d2h, dt, args.e2e_steps),
                        "path": "kernels.<op>(pinned numpy planes) per op -> "
                                "tf_elementwise_host (chunked H2D / kernel / D2H pipeline)"}}
    if not args.no_pageable:
        # the reference's callers pass plain numpy arrays (reference kernels.py:191-239,
        # bench.py:144-162): pageable planes, staged through pinned buffers until a
        # plane reused 4 times is page-locked in place (kernels._maybe_register)
        npg = min(ne, PAGEABLE_MAX)
        pcache = {}
        pcalls = []
        for op, hp in zip(ops, host_planes):
            pp = []
            for key, a in zip(ps.keys[op.name], hp):
                if key not in pcache:
                    pcache[key] = np.array(a[:npg], copy=True)
                pp.append(pcache[key])
            pcalls.append(pp)
        pout = K.TwofoldArray(np.empty(npg, host_out.value.dtype), np.empty(npg, host_out.value.dtype))
        pc = [_host_call_args(K, K.KERNELS[op.name].arity, pp, pout) for op, pp in zip(ops, pcalls)]
        barrier(world)
        times = []
        for _ in range(8):
            t0 = time.perf_counter()
            per_call_step(pc)
            times.append(time.perf_counter() - t0)
        first = max_over_ranks(times[0], world)
        steady = max_over_ranks(statistics.mean(times[5:]), world)
        u = len(ops) * npg
        locked = sum(1 for a in list(pcache.values()) + [pout.value, pout.error]
                     if a.ctypes.data in K._REG)
        rec["pageable"] = {"first_step": world * u / first, "steady_state": world * u / steady,
                           "step_s": times, "planes_page_locked": locked,
                           "planes": len(pcache) + 2,
                           "unit": "elem-ops/s", "elems_per_op": npg,
                           "h2d_bytes_per_step": sum(len(p) for p in pcalls) * esz * npg,
                           "d2h_bytes_per_step": 2 * esz * npg * len(ops),
                           "path": "kernels.<op>(plain numpy planes) per op: staged through "
                                   "pinned buffers; planes reused 4 times get page-locked "
                                   "(a plane read once per step locks during step 4; "
                                   "steady state = mean of steps 6-8)"}
        del pcache, pcalls, pout, pc
    return rec


def strong_elementwise(args, wlname, rank, world, local, n_total):
    """Strong-scaling record: ONE global array of n_total elements split into
    contiguous 32-byte-aligned slices (dist.shard_elementwise), same steps."""
    import torch

    from paper_1401_6235_b200 import dist as D

    wl = WL[wlname]
    esz = 8 if wl["dtype"] == np.float64 else 4
    lo, hi = D.shard_elementwise(n_total, world, rank, align=32 // esz)
    ops, ps, out = elementwise_ops(wlname, hi - lo, lo, torch.cuda.current_device())
    torch.cuda.synchronize()
    ws = sum(t.numel() * t.element_size() for t in ps.cache.values()) + 2 * (hi - lo) * esz
    tm = time_steps(args, ops, ws, world, local, hi - lo)
    rec = {"scaling": "strong", "n_total": n_total, "n_this_rank": hi - lo,
           "value": len(ops) * n_total * args.steps / (tm["elapsed_ms"] * 1e-3),
           "unit": "elem-ops/s", "ms_per_step": tm["elapsed_ms"] / args.steps,
           "per_op": tm["per_op"], "clocks": tm["clocks"],
           "how": "dist.shard_elementwise slices of one global array (no collective); "
                  "time = max over ranks"}
    del ops, ps, out
    return rec


def weak_elementwise_record(args, wlname, rank, world, local, n):
    """Weak-scaling record at N > 1 when the headline is strong (n per GPU)."""
    import torch

    wl = WL[wlname]
    esz = 8 if wl["dtype"] == np.float64 else 4
    ops, ps, out = elementwise_ops(wlname, n, rank * n, torch.cuda.current_device())
    torch.cuda.synchronize()
    ws = sum(t.numel() * t.element_size() for t in ps.cache.values()) + 2 * n * esz
    tm = time_steps(args, ops, ws, world, local, n)
    rec = {"scaling": "weak", "n_per_gpu": n,
           "value": world * len(ops) * n * args.steps / (tm["elapsed_ms"] * 1e-3),
           "unit": "elem-ops/s", "ms_per_step": tm["elapsed_ms"] / args.steps,
           "per_op": tm["per_op"], "clocks": tm["clocks"]}
    del ops, ps, out
    return rec


def run_elementwise(args, rank, world, local, wlname):
    import torch

    from paper_1401_6235_b200 import _lib

    wl = WL[wlname]
    dtype = wl["dtype"]
    esz = 8 if dtype == np.float64 else 4
    dts = "f64" if dtype == np.float64 else "f32"
    _lib.ensure_device(local)
    n_cfg = args.n or wl["n"]
    if args.scaling == "strong":
        from paper_1401_6235_b200 import dist as D

        lo, hi = D.shard_elementwise(n_cfg, world, rank, align=32 // esz)
    else:
        lo, hi = rank * n_cfg, (rank + 1) * n_cfg
    n = hi - lo
    log("%s: generating inputs n=%d (%s)" % (wlname, n, args.scaling))
    small = args.graph == "on" or (args.graph == "auto" and n <= (1 << 22))
    ops, ps, out = elementwise_ops(wlname, n, lo, torch.cuda.current_device(),
                                   separate_outputs=small and not args.serial_graph)
    torch.cuda.synchronize()
    ws_bytes = sum(t.numel() * t.element_size() for t in ps.cache.values()) + 2 * n * esz
    tm = time_steps(args, ops, ws_bytes, world, local, n)
    K = args.steps
    log("%s: timed region done: %.3f ms/step (graph=%s)" % (wlname, tm["elapsed_ms"] / K,
                                                            tm["use_graph"]))
    per_op = tm["per_op"]
    dom = max(per_op, key=lambda k: per_op[k]["ms"])
    peak, peak_src = measured_peak()
    units_per_step = len(ops) * n_cfg * (world if args.scaling == "weak" else 1)
    value = units_per_step * K / (tm["elapsed_ms"] * 1e-3)
    bytes_per_step = sum(op.nbytes for op in ops)
    dbatch, check = None, None
    if not args.no_device_batch and len(ops) > 1:
        log("%s: device batch" % wlname)
        dbatch, bouts = device_batch_leg(args, ops, n, esz, peak, world)
        check = ieee_check(ops, bouts)
        if rank == 0:
            check["oracle_sample"] = oracle_sample_check(ops, bouts)
            # the batch's bits equal one launch per op (the headline path): every
            # op whose output planes no later op overwrote, vs the batch's for it
            last = {id(op.out): j for j, op in enumerate(ops)}
            check["batch_equals_per_op_launch"] = {
                ops[j].name: bool(torch.equal(bouts[j].value, ops[j].out.value)
                                  and torch.equal(bouts[j].error, ops[j].out.error))
                for j in sorted(last.values())}
        del bouts
    e2e = None
    if not args.no_e2e:
        log("%s: e2e" % wlname)
        e2e = e2e_elementwise(args, ops, ps, n, esz, world, wlname)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        log("%s: cpu baseline" % wlname)
        ns = min(n, args.cpu_sample)

        def planes_of(name, ns=ns):  # the same inputs the GPU ran, first ns elements
            return [p[:ns].cpu().numpy() for p in ps.planes(name)]

        v, nt = cpu_baseline_elementwise(wl["names"], planes_of, ns)
        ns1 = min(ns, 1 << 23)  # one core: a smaller sample of the same planes
        v1, _ = cpu_baseline_elementwise(wl["names"], lambda name: [p[:ns1] for p in planes_of(name)],
                                         ns1, nthreads=1)
        cpu = {"value": v, "unit": "elem-ops/s", "cores": nt, "kind": "port",
               "sample": "first %d elements of the bench's own input planes per op over %s "
                         "(best of 3 per op), oracle/twofold_oracle.c OpenMP on %d threads"
                         % (ns, "/".join(wl["names"]), nt),
               "single_core": {"value": v1, "cores": 1, "sample": "first %d elements per op" % ns1}}
    del ops, ps, out
    other = None
    if world > 1 and not args.no_other_scaling:
        release_memory()
        log("%s: other scaling mode" % wlname)
        other = (strong_elementwise(args, wlname, rank, world, local, n_cfg)
                 if args.scaling == "weak" else
                 weak_elementwise_record(args, wlname, rank, world, local, n_cfg))
    if rank != 0:
        return None
    d = per_op[dom]
    step_gbs = world * bytes_per_step * K / (tm["elapsed_ms"] * 1e-3) / 1e9
    return {
        "metric": METRIC if wlname == "config2" else METRIC + " [%s]" % wlname,
        "value": value, "unit": "elem-ops/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": tm["elapsed_ms"] / K,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": dts,
        "data": "synthetic (seeded, device-generated with BASELINE distributions)",
        "config": wl_config(wlname, n_cfg, args.scaling),
        "config_detail": {
            "timing": ("cuda-graph replay per step" + (
                "; the ops are independent (each its own output planes) and run as parallel "
                "graph branches" if tm["graph_branches"] else "")) if tm["use_graph"]
            else "eager launches",
            "l2_flush": tm["flush"], "layout": "split SoA planes",
            "inputs": "tf_fill counter-based splitmix64 on the device; plane k seed 1000+17k, "
                      "element i of a rank is global index lo+i",
            "l2": ("working set %d MiB < L2 x3: flushed" if tm["flush"] else
                   "working set %d MiB >> 126 MB L2; no flush") % (ws_bytes >> 20),
            "n_this_rank": n},
        "hbm_gbs": step_gbs,
        "roofline": dict(
            {"bound": "hbm", "kernel": dom, "achieved": d["gbs"], "peak": peak,
             "unit": "GB/s", "frac": d["gbs"] / peak,
             "traffic": ncu_traffic(dom, dts, n),
             "algorithmic_bytes": d["bytes"], "peak_source": peak_src},
            # launch-bound steps: `achieved` is one launch alone (events around an eager
            # launch, their latency included); the whole step's bytes over the step's
            # time — the concurrent graph branches together — is the rate HBM saw
            **({"step": {"achieved": step_gbs / world, "frac": step_gbs / world / peak,
                         "what": "all launches of one graph replay, bytes / step time"}}
               if tm["use_graph"] else {})),
        "per_op": per_op,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "device_batch": dbatch,
        "check": check,
        "other_scaling": other,
        "gpu_launches": tm["launches"] * world,
        "clocks": tm["clocks"],
    }


# --------------------------------------------------------------------------
# config 4: ill-conditioned dot + sum (reductions with one cross-GPU exchange)


def _golden_config4():
    p = ROOT / "tests" / "golden" / "config4.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


def _bits_of(z):
    return [float(z[0]).hex(), float(z[1]).hex()]


def exact_check(problems, results, nt):
    """Results against the oracle's exact integer-limb accumulator: achieved
    condition numbers and the north star's bound |(z0+z1) - exact| <= 4u Σ|terms|
    (u = 2^-53).  problems: {"vtdot": (x, y), "vtsum": (p,)}; results: name ->
    (z0, z1)."""
    from fractions import Fraction

    from oracle import oracle as o

    u4 = 4 * Fraction(1, 2**53)
    out = {}
    for name, planes in problems.items():
        rop = "dot" if name == "vtdot" else "sum"
        z = results[name]
        s, t = o.exact(rop, *planes, nthreads=nt)
        err = abs(Fraction(float(z[0])) + Fraction(float(z[1])) - s)
        out[name] = {"cond": float((2 if rop == "dot" else 1) * t / abs(s)) if s else float("inf"),
                     "cond1": float(t / abs(s)) if s else float("inf"),
                     "bound_ok": bool(err <= u4 * t),
                     "err_over_bound": float(err / (u4 * t)) if t else 0.0,
                     "z0_rel_err": float(abs(Fraction(float(z[0])) - s) / abs(s)) if s else None,
                     "z0_plus_z1_rel_err": float(err / abs(s)) if s else None}
    out["how"] = ("oracle exact accumulator (integer limbs, exact 106-bit products) over all "
                  "%d elements; cond(dot) = 2*sum|x*y|/|sum x*y| (Ogita-Rump-Oishi), cond1(dot) "
                  "= sum|x*y|/|sum x*y|, cond(sum) = cond1(sum) = sum|p|/|sum p|"
                  % len(next(iter(problems.values()))[0]))
    return out


def config4_exchange(part, counts, world, res):
    """The one exchange step: every rank's (2, 2) partials (dot row, sum row) in
    ONE all-gather (NCCL over NVLink), then the adjacent-pair _tadd tree over
    ranks for each reduction (tf_combine) into res."""
    from paper_1401_6235_b200 import dist as D, reduce as R

    allp = D.gather_partials(part)  # (world, 2, 2)
    R.combine(allp[:, 0].contiguous(), counts, out=res[0])
    R.combine(allp[:, 1].contiguous(), counts, out=res[1])


def config4_timed(args, X, Y, P, counts, world, local, tp=None):
    """K steps of vtdot(X, Y) + vtsum(P) (+ the exchange at N > 1); events around
    the local reductions and the exchange separately."""
    import torch

    from paper_1401_6235_b200 import reduce as R

    part = torch.empty((2, 2), dtype=torch.float64, device="cuda")
    res = torch.empty((2, 2), dtype=torch.float64, device="cuda")

    def local_red():
        if tp is not None:  # reduction + NVLink exchange fused in one launch, no NCCL
            tp.reduce("dot", (X, Y), counts, out=res[0])
            tp.reduce("sum", (P,), counts, out=res[1])
            return
        R.vtdot(X, Y, out=part[0])
        R.vtsum(P, out=part[1])

    def exchange():
        if tp is not None:
            return
        if world > 1:
            config4_exchange(part, counts, world, res)
        else:
            res.copy_(part)

    for _ in range(args.warmup):
        local_red()
        exchange()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record(stream)
        for s in range(K):
            ev[s][0].record(stream)
            if tp is None:
                R.vtdot(X, Y, out=part[0])
                ev[s][1].record(stream)
                R.vtsum(P, out=part[1])
            else:
                tp.reduce("dot", (X, Y), counts, out=res[0])
                ev[s][1].record(stream)
                tp.reduce("sum", (P,), counts, out=res[1])
            ev[s][2].record(stream)
            exchange()
            ev[s][3].record(stream)
        end.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    elapsed = max_over_ranks(start.elapsed_time(end), world)
    dot_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / K
    sum_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / K
    xch_ms = sum(e[2].elapsed_time(e[3]) for e in ev) / K
    return {"elapsed_ms": elapsed, "dot_ms": dot_ms, "sum_ms": sum_ms, "exchange_ms": xch_ms,
            "part": part, "res": res, "clocks": clk.summary()}


def run_config4(args, rank, world, local):
    """f64 vtdot(x, y) + vtsum(p) over config 4's ill-conditioned planes: every
    rank generates its shard_tiles slice of ONE global problem (blocked
    generator, csrc/gen_ill.cu), reduces it in the canonical order, and the
    partials meet in one all-gather + tf_combine."""
    import torch

    from paper_1401_6235_b200 import _lib, dist as D, reduce as R, workloads as WLs

    wl = WL["config4"]
    n_cfg = args.n or wl["n"]
    L = WLs.GEN_BLOCK
    _lib.ensure_device(local)
    assert R.tile_elems(np.float64) == L
    n_glob = n_cfg * world if args.scaling == "weak" else n_cfg
    lo, hi = D.shard_tiles(n_glob, world, rank, L)
    counts = D.shard_counts(n_glob, world, L)
    if min(counts) <= 0:
        raise SystemExit("config4: %d elements leave a rank without a whole tile (counts %s)"
                         % (n_glob, counts))
    n = hi - lo
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    X, Y, P = WLs.config4_planes(n_glob, lo, n, torch.cuda.current_device())
    g1.record()
    torch.cuda.synchronize()
    gen_ms = g0.elapsed_time(g1)
    log("config4: generated %d of %d elements on the device in %.1f ms" % (n, n_glob, gen_ms))
    tp = D.P2PTransport() if args.reduce_transport == "p2p" else None
    tm = config4_timed(args, X, Y, P, counts, world, local, tp)
    K = args.steps
    peak, src = measured_peak()
    value = 2 * n_glob * K / (tm["elapsed_ms"] * 1e-3)
    zdot = tm["res"][0].cpu().tolist()
    zsum = tm["res"][1].cpu().tolist()
    local_bits = {"vtdot": _bits_of(tm["part"][0].cpu().tolist()),
                  "vtsum": _bits_of(tm["part"][1].cpu().tolist())}
    golden = _golden_config4()
    check = {"result": {"vtdot": _bits_of(zdot), "vtsum": _bits_of(zsum)}}
    if golden is not None:
        gp = golden["prefixes"]
        if str(n_glob) in gp:
            g = gp[str(n_glob)]
            check["golden_bits_equal"] = {nm: check["result"][nm] == [g[nm]["z0"], g[nm]["z1"]]
                                          for nm in ("vtdot", "vtsum")}
        if world > 1 and rank == 0 and tp is None and str(n) in gp:
            # rank 0's shard is the first n elements of the global problem, a
            # complete subtree: its local result is the N = 1 result of that prefix
            g = gp[str(n)]
            check["rank0_local_equals_n1_golden"] = {
                nm: local_bits[nm] == [g[nm]["z0"], g[nm]["z1"]] for nm in ("vtdot", "vtsum")}
        check["golden"] = "tests/golden/config4.json (oracle canonical order over the host generator's planes, make_config4_golden.py)"
    # e2e: the public API on host planes (bounded sample of this rank's planes)
    e2e = None
    ne = min(n, E2E_MAX)
    xh = yh = ph = None
    if not args.no_e2e:
        log("config4: e2e")
        xh, yh, ph = _pinned_copy(X[:ne]), _pinned_copy(Y[:ne]), _pinned_copy(P[:ne])
        R.host_batch([("vtdot", xh, yh), ("vtsum", ph)])
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            R.host_batch([("vtdot", xh, yh), ("vtsum", ph)])
        dtb = max_over_ranks(time.perf_counter() - t0, world)
        R.vtdot(xh, yh)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            R.vtdot(xh, yh)
            R.vtsum(ph)
        dt = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": world * 2 * ne * args.e2e_steps / dtb, "unit": "elem-ops/s",
               "elems_per_step": ne, "h2d_bytes_per_step": 24 * ne, "d2h_bytes_per_step": 32,
               "roofline": link_roofline(24 * ne, 32, dtb, args.e2e_steps),
               "path": "reduce.host_batch([vtdot(x, y), vtsum(p)]) on pinned numpy planes -> "
                       "tf_reduce_host_batch (one chunked H2D pass, on-device canonical trees)",
               "per_call": {"value": world * 2 * ne * args.e2e_steps / dt,
                            "path": "reduce.vtdot / reduce.vtsum on pinned numpy planes -> "
                                    "tf_reduce_host"}}
        if not args.no_pageable:
            npg = min(ne, PAGEABLE_MAX)
            xp, yp, pp = (np.array(a[:npg], copy=True) for a in (xh, yh, ph))
            times = []
            for _ in range(8):
                t0 = time.perf_counter()
                R.vtdot(xp, yp)
                R.vtsum(pp)
                times.append(time.perf_counter() - t0)
            e2e["pageable"] = {"first_step": world * 2 * npg / max_over_ranks(times[0], world),
                               "steady_state": world * 2 * npg /
                               max_over_ranks(statistics.mean(times[5:]), world),
                               "unit": "elem-ops/s", "elems_per_step": npg,
                               "path": "reduce.vtdot / vtsum on plain numpy planes (staged; "
                                       "page-locked after 4 uses; steady = steps 6-8)"}
            del xp, yp, pp
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as o

        log("config4: cpu baseline")
        nt = os.cpu_count() or 1
        ns = min(n, args.cpu_sample)
        xs, ys, ps_ = (t[:ns].cpu().numpy() for t in (X, Y, P))
        t_dot = _best_of(lambda: o.reduce("dot", xs, ys, geometry=(2, 256, 128), nthreads=nt))
        t_sum = _best_of(lambda: o.reduce("sum", ps_, geometry=(2, 256, 128), nthreads=nt))
        cpu = {"value": 2 * ns / (t_dot + t_sum), "unit": "elem-ops/s", "cores": nt, "kind": "port",
               "sample": "first %d elements of the bench's own planes, vtdot(x, y) + vtsum(p) "
                         "(best of 3 each), oracle/twofold_oracle.c canonical order, OpenMP on "
                         "%d threads" % (ns, nt)}
        del xs, ys, ps_
    if rank == 0 and world == 1 and not args.no_check:
        from oracle import oracle as o

        log("config4: full-size check: oracle canonical order + exact accumulator")
        nt = os.cpu_count() or 1
        xf, yf, pf = (t.cpu().numpy() for t in (X, Y, P))
        wd = o.reduce("dot", xf, yf, geometry=(2, 256, 128), nthreads=nt)
        wsm = o.reduce("sum", pf, geometry=(2, 256, 128), nthreads=nt)
        check["bit_exact_vs_oracle"] = {"vtdot": _bits_of(wd) == check["result"]["vtdot"],
                                        "vtsum": _bits_of(wsm) == check["result"]["vtsum"]}
        check["exact"] = exact_check({"vtdot": (xf, yf), "vtsum": (pf,)},
                                     {"vtdot": zdot, "vtsum": zsum}, nt)
        del xf, yf, pf
    del X, Y, P, xh, yh, ph
    other = None
    if world > 1 and not args.no_other_scaling:
        release_memory()
        other = config4_other_scaling(args, rank, world, local, n_cfg, tp)
    if rank != 0:
        return None
    dgbs = 16 * n / (tm["dot_ms"] * 1e-3) / 1e9
    sgbs = 8 * n / (tm["sum_ms"] * 1e-3) / 1e9
    return {
        "metric": METRIC + " [config4: vtdot+vtsum]", "value": value, "unit": "elem-ops/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": tm["elapsed_ms"] / K,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (blocked ORO-style ill-conditioned dot and sum, cond 1e16, exponents "
                "in [-50, 50], seeded, device-generated)",
        "config": wl_config("config4", n_cfg, args.scaling),
        "config_detail": {"n_global": n_glob, "n_this_rank": n, "counts": counts,
                          "generator_ms": gen_ms,
                          "generator": "tf_gen_ill (csrc/gen_ill.cu): per 65536-element block, "
                                       "half the terms random with exponents in [-50, 50], the "
                                       "rest cancel the running value; calibrated to cond 1e16"},
        "roofline": {"bound": "hbm", "kernel": "vtdot", "achieved": dgbs, "peak": peak,
                     "unit": "GB/s", "frac": dgbs / peak, "traffic": ncu_traffic("vtdot", "f64", n),
                     "algorithmic_bytes": 16 * n, "peak_source": src,
                     "vtsum": {"achieved": sgbs, "frac": sgbs / peak, "algorithmic_bytes": 8 * n,
                               "traffic": ncu_traffic("vtsum", "f64", n)}},
        "per_op": {"vtdot": {"ms": tm["dot_ms"], "gbs": dgbs},
                   "vtsum": {"ms": tm["sum_ms"], "gbs": sgbs},
                   "exchange": {"ms": tm["exchange_ms"],
                                "what": ("one NCCL all_gather_into_tensor of the (2, 2) partials + "
                                         "2 tf_combine launches" if world > 1 and tp is None else
                                         "fused into the reductions (p2p)" if tp is not None
                                         else "device copy of the partials (1 GPU)")}},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "check": check,
        "other_scaling": other,
        "gpu_launches": world * K * (2 + (2 if world > 1 and tp is None else 0)),
        "reduce_transport": (args.reduce_transport if world > 1 else
                             "p2p (fused reduce + mailbox exchange, 1 rank)" if tp is not None
                             else "none (1 GPU)"),
        "clocks": tm["clocks"],
    }


def config4_other_scaling(args, rank, world, local, n_cfg, tp):
    """At N > 1: the other scaling mode.  For the strong record (ONE problem of
    n_cfg elements split over the ranks) rank 0 also reduces the whole problem
    alone — the N = 1 result — and the record asserts the bits are equal."""
    import torch

    from paper_1401_6235_b200 import dist as D, reduce as R, workloads as WLs

    L = WLs.GEN_BLOCK
    mode = "strong" if args.scaling == "weak" else "weak"
    n_glob = n_cfg if mode == "strong" else n_cfg * world
    ref_bits = None
    if mode == "strong" and rank == 0:
        # the N = 1 reference: the whole problem on this one GPU
        X1, Y1, P1 = WLs.config4_planes(n_glob, 0, n_glob, torch.cuda.current_device())
        z = torch.empty((2, 2), dtype=torch.float64, device="cuda")
        R.vtdot(X1, Y1, out=z[0])
        R.vtsum(P1, out=z[1])
        zz = z.cpu().tolist()
        ref_bits = {"vtdot": _bits_of(zz[0]), "vtsum": _bits_of(zz[1])}
        del X1, Y1, P1, z
        release_memory()
    barrier(world)
    lo, hi = D.shard_tiles(n_glob, world, rank, L)
    counts = D.shard_counts(n_glob, world, L)
    if min(counts) <= 0:
        return {"scaling": mode, "skipped": "%d elements leave a rank without a tile" % n_glob}
    X, Y, P = WLs.config4_planes(n_glob, lo, hi - lo, torch.cuda.current_device())
    torch.cuda.synchronize()
    a2 = copy.copy(args)
    a2.steps = max(3, min(args.steps, args.sub_steps))
    tm = config4_timed(a2, X, Y, P, counts, world, local, tp)
    res = tm["res"].cpu().tolist()
    bits = {"vtdot": _bits_of(res[0]), "vtsum": _bits_of(res[1])}
    rec = {"scaling": mode, ("n_total" if mode == "strong" else "n_per_gpu"): n_cfg,
           "n_global": n_glob, "counts": counts,
           "value": 2 * n_glob * a2.steps / (tm["elapsed_ms"] * 1e-3), "unit": "elem-ops/s",
           "ms_per_step": tm["elapsed_ms"] / a2.steps, "steps": a2.steps,
           "exchange_ms": tm["exchange_ms"], "result": bits}
    if ref_bits is not None:
        rec["n1_result"] = ref_bits
        rec["same_bits_as_n1"] = ref_bits == bits
    g = _golden_config4()
    if g is not None and str(n_glob) in g["prefixes"]:
        gg = g["prefixes"][str(n_glob)]
        rec["golden_bits_equal"] = {nm: bits[nm] == [gg[nm]["z0"], gg[nm]["z1"]]
                                    for nm in ("vtdot", "vtsum")}
    del X, Y, P
    return rec


# --------------------------------------------------------------------------
# config 5: twofold Horner (FP64-pipe bound)


def horner_timed(args, x, out, c, world, local):
    import torch

    from paper_1401_6235_b200 import reduce as R

    for _ in range(args.warmup):
        R.vthorner(c, x, out)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record(stream)
        for _ in range(args.steps):
            R.vthorner(c, x, out)
        end.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(start.elapsed_time(end), world), clk.summary()


def run_config5(args, rank, world, local):
    """f64 twofold Horner of the expanded (x-1)^20 at n = 2^26 points per GPU."""
    import ctypes

    import torch

    from paper_1401_6235_b200 import _lib, dist as D, kernels as Kmod, reduce as R
    from paper_1401_6235_b200 import workloads as WLs

    n_cfg = args.n or WL["config5"]["n"]
    if args.scaling == "strong":
        lo, hi = D.shard_elementwise(n_cfg, world, rank, align=4)
    else:
        lo, hi = rank * n_cfg, (rank + 1) * n_cfg
    n = hi - lo
    _lib.ensure_device(local)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    WLs.fill(x, WLs.UNIFORM, 555, lo, 0.9, 1.1)
    out = Kmod.empty_twofold(n, torch.float64)
    c = R.binomial_coeffs(20)
    pi, pm = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib().tf_fp64_peak(local, ctypes.byref(pi), ctypes.byref(pm)), "fp64_peak")
    fp64_peak = pi.value / (pm.value * 1e-3)
    elapsed_ms, clocks = horner_timed(args, x, out, c, world, local)
    K = args.steps
    per_ms = elapsed_ms / K
    instr = 220.0 * n
    achieved = instr / (per_ms * 1e-3)
    value = (world * n_cfg if args.scaling == "weak" else n_cfg) * K / (elapsed_ms * 1e-3)
    # full-size property check of the timed run's own outputs, on the device:
    # (x-1)^20 evaluated stably (x-1 is exact for x in [0.5, 2], then 20 ulps at
    # most) against the expanded-polynomial Horner; z1 must flag the cancellation
    with torch.no_grad():
        p = (x - 1.0).pow(20)
        z0, z1 = out.value, out.error
        nz = (z0 != 0) & (p != 0)
        flagged = ((z1.abs() >= 0.5 * z0.abs()) & nz).sum().item()
        rel0 = ((z0 - p).abs() / p.abs())[nz]
        rel01 = (((z0 + z1) - p).abs() / p.abs())[nz]
        check = {"points": n, "nonzero": int(nz.sum().item()),
                 "flag_rate": flagged / max(1, int(nz.sum().item())),
                 "median_rel_err_z0": rel0.median().item(),
                 "median_rel_err_z0_plus_z1": rel01.median().item(),
                 "how": "on the device: reference (x-1)^20 by torch.pow of the exact x-1; "
                        "flag = |z1| >= 0.5|z0| where z0 != 0"}
        del p, nz, rel0, rel01
    if rank == 0:
        from oracle import oracle as o

        k = min(n, 1 << 20)
        xs = x[:k].cpu().numpy()
        h0, h1 = o.horner(c, xs)
        g0, g1 = out.value[:k].cpu().numpy(), out.error[:k].cpu().numpy()
        check["oracle_sample"] = {
            "bit_exact_vs_oracle": bool(np.array_equal(g0.view(np.uint64), h0.view(np.uint64))
                                        and np.array_equal(g1.view(np.uint64), h1.view(np.uint64))),
            "elements": k}
    # e2e: the public API on host planes (tf_horner_host pipeline)
    e2e = None
    ne = min(n, E2E_MAX)
    xh = None
    if not args.no_e2e:
        xh = _pinned_copy(x[:ne])
        oh = Kmod.empty_twofold(ne, np.float64, pin_memory=True)
        R.vthorner(c, xh, oh)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            R.vthorner(c, xh, oh)
        dte = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": world * ne * args.e2e_steps / dte, "unit": "points/s",
               "h2d_bytes_per_step": 8 * ne, "d2h_bytes_per_step": 16 * ne,
               "elems_per_step": ne,
               "roofline": link_roofline(8 * ne, 16 * ne, dte, args.e2e_steps),
               "path": "reduce.vthorner on pinned numpy planes -> tf_horner_host"}
        if not args.no_pageable:
            npg = min(ne, PAGEABLE_MAX)
            xp = np.array(xh[:npg], copy=True)
            op_ = Kmod.empty_twofold(npg)  # numpy planes (the reference's default)
            times = []
            for _ in range(8):
                t0 = time.perf_counter()
                R.vthorner(c, xp, op_)
                times.append(time.perf_counter() - t0)
            e2e["pageable"] = {"first_step": world * npg / max_over_ranks(times[0], world),
                               "steady_state": world * npg /
                               max_over_ranks(statistics.mean(times[5:]), world),
                               "unit": "points/s", "elems_per_step": npg,
                               "path": "reduce.vthorner on plain numpy planes (staged; "
                                       "page-locked after 4 uses; steady = steps 6-8)"}
            del xp, op_
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as o

        nt = os.cpu_count() or 1
        ns = min(n, args.cpu_sample, 1 << 24)
        xs = x[:ns].cpu().numpy()
        oo = (np.zeros_like(xs), np.zeros_like(xs))
        t = _best_of(lambda: o.horner(c, xs, nthreads=nt, out=oo))
        cpu = {"value": ns / t, "unit": "points/s", "cores": nt, "kind": "port",
               "sample": "first %d of the bench's own points (best of 3), oracle/twofold_oracle.c "
                         "OpenMP on %d threads" % (ns, nt)}
    del x, out, xh
    other = None
    if world > 1 and not args.no_other_scaling:
        release_memory()
        mode = "strong" if args.scaling == "weak" else "weak"
        lo2, hi2 = (D.shard_elementwise(n_cfg, world, rank, align=4) if mode == "strong"
                    else (rank * n_cfg, (rank + 1) * n_cfg))
        x2 = torch.empty(hi2 - lo2, dtype=torch.float64, device="cuda")
        WLs.fill(x2, WLs.UNIFORM, 555, lo2, 0.9, 1.1)
        o2 = Kmod.empty_twofold(hi2 - lo2, torch.float64)
        ms2, clk2 = horner_timed(args, x2, o2, c, world, local)
        tot = n_cfg if mode == "strong" else n_cfg * world
        other = {"scaling": mode, "n_global": tot, "value": tot * K / (ms2 * 1e-3),
                 "unit": "points/s", "ms_per_step": ms2 / K, "clocks": clk2}
        del x2, o2
    if rank != 0:
        return None
    nominal = fp64_nominal(clocks.get("sm_max_mhz") or 1965.0)
    return {
        "metric": METRIC + " [config5: twofold Horner points/s, (x-1)^20]", "value": value,
        "unit": "points/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": per_ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic x ~ U[0.9,1.1] (seeded, device-generated)",
        "config": wl_config("config5", n_cfg, args.scaling),
        "roofline": {"bound": "fp64", "kernel": "vthorner", "achieved": achieved / 1e12,
                     "peak": fp64_peak / 1e12, "unit": "T FP64 instr/s",
                     "frac": achieved / fp64_peak, "traffic": ncu_traffic("vthorner", "f64", n),
                     "algorithmic_instr": instr,
                     "peak_source": "measured live: tf_fp64_peak (independent DFMA chains); "
                                    "MEASURED_PEAKS.json has no FP64 figure",
                     "nominal_peak": nominal / 1e12, "frac_of_nominal": achieved / nominal,
                     "nominal_source": "148 SMs x 64 FP64 instr/clk x sm_max_mhz"},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "check": check,
        "other_scaling": other,
        "gpu_launches": world * K,
        "clocks": clocks,
    }


# --------------------------------------------------------------------------
# reference arm: the reference algorithm's CPU implementation (the oracle port)


def _reference_line(args, wlname, metric, value, unit, dtype, n_cfg, sample, nt, steps, ms,
                    **extra):
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit,
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (seeded numpy / host generator, BASELINE distributions)",
        "config": wl_config(wlname, n_cfg, args.scaling),
        "cpu_baseline": {"value": value, "unit": unit, "cores": nt, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    line.update(extra)
    return line


def _timed_steps(steps, warmup, step, warm_s=1.0):
    t0 = time.perf_counter()
    k = 0
    while k < max(warmup, 1) or time.perf_counter() - t0 < warm_s:  # also warms the CPUs
        step()
        k += 1
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    return time.perf_counter() - t0


def reference_elementwise(args, wlname, steps):
    from oracle import oracle as o

    wl = WL[wlname]
    n_cfg = args.n or wl["n"]
    esz = 8 if wl["dtype"] == np.float64 else 4
    # full size where host RAM allows (shared input planes + 2 output planes)
    need = (REF_PLANES[wlname] + 2) * esz * n_cfg
    ns = args.ref_elems or (n_cfg if need < 0.4 * host_ram_available() else min(n_cfg, 1 << 26))
    inputs = ref_planes(wlname, ns)
    nt = os.cpu_count() or 1
    out = (np.zeros(ns, wl["dtype"]), np.zeros(ns, wl["dtype"]))

    def step():
        for name in wl["names"]:
            o.elementwise(name, *inputs[name], nthreads=nt, out=out)

    dt = _timed_steps(steps, args.warmup, step)
    value = len(wl["names"]) * ns * steps / dt
    sample = ("%s %d elements per op x %d ops per step, oracle/twofold_oracle.c (OpenMP, -O3 "
              "-march=x86-64-v3, no contraction)"
              % ("all" if ns == n_cfg else "a sample of", ns, len(wl["names"])))
    del out
    port = {"value": value, "cores": nt, "sample": sample, "ms_per_step": 1e3 * dt / steps}
    numba = None
    if not args.no_numba_ref:
        gc.collect()
        try:
            numba = _numba_reference_timing(wlname, inputs, ns, steps, args.warmup)
        except Exception as e:  # noqa: BLE001
            numba = {"unavailable": "%s: %s" % (type(e).__name__, e)}
    del inputs
    # the arm's value is the STRONGER of the two CPU implementations on this box:
    # the reference package itself (numba, fork-sharded) or the 16-thread C port
    kind = "port"
    if numba and "value" in numba and numba["value"] > value:
        kind, value, nt = "reference", numba["value"], numba["cores"]
        sample = numba["sample"] + ", " + numba["code"]
    line = _reference_line(args, wlname, METRIC if wlname == "config2" else METRIC + " [%s]" % wlname,
                           value, "elem-ops/s",
                           "f64" if wl["dtype"] == np.float64 else "f32", n_cfg, sample, nt,
                           steps, 1e3 * len(wl["names"]) * ns / value, sample_elems_per_op=ns,
                           port=port, numba_reference=numba)
    line["cpu_baseline"]["kind"] = kind
    return line


def _numba_reference_timing(wlname, inputs, ns, steps, warmup):
    """The reference package itself (twofold.kernels, numba, staged unmodified in
    baseline/_ref) on the same planes as the port leg, as BASELINE.md §5 plans it:
    KERNELS[name].func on numpy planes, fork-sharded over all host cores in
    contiguous slices (the numba loops hold the GIL, so threads do not scale),
    warm-up steps first (numba compile, page faults), then `steps` timed steps of
    every op between two barriers; throughput = elements / slowest process.  P = 1
    is timed too (one step).  None when the staged package or numba is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "twofold").is_dir():
        return None
    try:
        import multiprocessing as mp

        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tf_numba_cache")
        sys.path.insert(0, str(ref))
        import twofold.kernels as RK  # the reference's own module
    except Exception as e:  # noqa: BLE001
        return {"unavailable": "%s: %s" % (type(e).__name__, e)}
    finally:
        if sys.path and sys.path[0] == str(ref):
            sys.path.pop(0)
    wl = WL[wlname]

    def step(lo, hi, out):
        for name in wl["names"]:
            spec = RK.KERNELS[name]
            pl = [q[lo:hi] for q in inputs[name]]
            if spec.arity == "22":
                spec.func(RK.TwofoldArray(pl[0], pl[1]), RK.TwofoldArray(pl[2], pl[3]), out)
            elif spec.arity == "21":
                spec.func(RK.TwofoldArray(pl[0], pl[1]), pl[2], out)
            elif spec.arity == "u2":
                spec.func(RK.TwofoldArray(pl[0], pl[1]), out)
            else:
                spec.func(*pl, out)

    n1 = min(ns, 1 << 24)  # the single-process figure on a bounded sample
    out1 = RK.empty_twofold(n1, wl["dtype"])
    step(0, n1, out1)  # compile
    t0 = time.perf_counter()
    step(0, n1, out1)
    t1 = time.perf_counter() - t0
    del out1
    p = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    limit = 900.0  # a wedged or killed child must not hang the bench
    bar = ctx.Barrier(p + 1, timeout=limit)
    q = ctx.Queue()

    def child(r):
        lo, hi = ns * r // p, ns * (r + 1) // p
        out = RK.empty_twofold(hi - lo, wl["dtype"])
        for _ in range(max(1, warmup)):
            step(lo, hi, out)
        bar.wait()
        t0 = time.perf_counter()
        for _ in range(steps):
            step(lo, hi, out)
        q.put(time.perf_counter() - t0)
        bar.wait()

    procs = [ctx.Process(target=child, args=(r,), daemon=True) for r in range(p)]
    for pr in procs:
        pr.start()
    try:
        bar.wait()
        bar.wait()
        tp = max(q.get(timeout=limit) for _ in procs)
    finally:
        for pr in procs:
            pr.join(timeout=5)
            if pr.is_alive():
                pr.terminate()
    nops = len(wl["names"])
    return {"value": nops * ns * steps / tp, "unit": "elem-ops/s", "cores": p,
            "sample": "%d elements per op x %d ops per step (%s), %d steps after %d warm-up, "
                      "the port leg's planes" % (ns, nops, "/".join(wl["names"]), steps,
                                                 max(1, warmup), ),
            "how": "fork-sharded contiguous slices over all host cores, barrier before and "
                   "after the timed steps, elements / slowest process",
            "single_process": {"value": nops * n1 / t1, "cores": 1, "steps": 1,
                               "elems_per_op": n1},
            "code": "baseline/_ref/twofold/kernels.py KERNELS[name].func (numba %s)"
                    % _numba_version()}


def _numba_version():
    try:
        import numba

        return numba.__version__
    except Exception:  # noqa: BLE001
        return "?"



def reference_config4(args, steps):
    """The oracle's canonical-order vtdot + vtsum on all host threads over the
    config-4 planes (tf_gen_ill_host: the same bits the device generator makes)."""
    from oracle import oracle as o
    from paper_1401_6235_b200 import workloads as WLs

    n_cfg = args.n or WL["config4"]["n"]
    ns = args.ref_elems or min(n_cfg, 1 << 26)
    ns = max(WLs.GEN_BLOCK, ns - ns % WLs.GEN_BLOCK) if ns >= WLs.GEN_BLOCK else ns
    x, y, p = np.empty(ns), np.empty(ns), np.empty(ns)
    WLs.gen_ill(WLs.GEN_DOT, x, y, n_total=n_cfg)
    WLs.gen_ill(WLs.GEN_SUM, p, n_total=n_cfg)
    nt = os.cpu_count() or 1

    def step():
        o.reduce("dot", x, y, geometry=(2, 256, 128), nthreads=nt)
        o.reduce("sum", p, geometry=(2, 256, 128), nthreads=nt)

    dt = _timed_steps(steps, args.warmup, step)
    value = 2 * ns * steps / dt
    return _reference_line(
        args, "config4", METRIC + " [config4: vtdot+vtsum]", value, "elem-ops/s", "f64", n_cfg,
        "first %d elements of the config-4 problem per step (vtdot(x, y) + vtsum(p)), "
        "oracle/twofold_oracle.c canonical order, OpenMP over tiles" % ns, nt, steps,
        1e3 * dt / steps, sample_elems_per_op=ns)


def reference_config5(args, steps):
    """The oracle's twofold Horner of (x-1)^20, all host threads."""
    import math

    from oracle import oracle as o

    n_cfg = args.n or WL["config5"]["n"]
    ns = args.ref_elems or min(n_cfg, 1 << 24)
    x = np.random.default_rng(555).uniform(0.9, 1.1, ns)
    c = [float((-1) ** (20 - k) * math.comb(20, k)) for k in range(21)]
    nt = os.cpu_count() or 1
    out = (np.zeros_like(x), np.zeros_like(x))
    dt = _timed_steps(steps, args.warmup, lambda: o.horner(c, x, nthreads=nt, out=out))
    value = ns * steps / dt
    return _reference_line(
        args, "config5", METRIC + " [config5: twofold Horner points/s, (x-1)^20]", value,
        "points/s", "f64", n_cfg,
        "%d points x ~ U[0.9,1.1] per step, oracle/twofold_oracle.c OpenMP" % ns, nt, steps,
        1e3 * dt / steps, sample_elems_per_op=ns)


def run_reference_workload(args, wlname, steps):
    if wlname == "config4":
        return reference_config4(args, steps)
    if wlname == "config5":
        return reference_config5(args, steps)
    return reference_elementwise(args, wlname, steps)


def run_reference(args, rank, world):
    """CPU reference arm: the oracle port on all host threads (rank 0 only)."""
    if rank != 0:
        return 0
    line = run_reference_workload(args, args.workload, args.steps)
    if args.workload == "config2" and not args.no_sub_workloads:
        subs = {}
        for wl in SUB_WORKLOADS:
            a2 = copy.copy(args)
            a2.n = args.sub_elems
            a2.warmup = min(args.warmup, 2)
            subs[wl] = run_reference_workload(a2, wl, max(1, min(args.steps, args.sub_steps)))
            gc.collect()
        line["workloads"] = subs
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------


def run_workload(args, wlname, rank, world, local):
    if wlname == "config4":
        return run_config4(args, rank, world, local)
    if wlname == "config5":
        return run_config5(args, rank, world, local)
    return run_elementwise(args, rank, world, local, wlname)


def main(argv=None):
    global E2E_MAX, PAGEABLE_MAX
    args = parse(argv)
    rank, world, local = env_rank()
    if world > 1:  # ranks of one node share its host memory: 0.5 GiB host planes
        E2E_MAX = 1 << 26
        PAGEABLE_MAX = 1 << 25
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch

    if os.environ.get("BENCH_DIST_BACKEND", "nccl") != "nccl":
        local = 0  # dry run: every rank on cuda:0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        # BENCH_DIST_BACKEND=gloo: host-side dry run of the multi-rank path on one
        # GPU (no kernel waits on another rank; never used for reported numbers)
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    try:
        line = run_workload(args, args.workload, rank, world, local)
        if args.workload == "config2" and not args.no_sub_workloads:
            subs = {}
            for wl in SUB_WORKLOADS:
                release_memory()
                a2 = copy.copy(args)
                a2.n = args.sub_elems
                a2.steps = max(1, min(args.steps, args.sub_steps))
                if wl == "config1":  # 16 us steps: five times as many for a steadier mean
                    a2.steps = min(5 * a2.steps, 50)
                a2.warmup = max(3, min(args.warmup, 3))
                a2.e2e_steps = 1
                a2.cpu_sample = min(args.cpu_sample, 1 << 24)
                log("sub-workload %s" % wl)
                rec = run_workload(a2, wl, rank, world, local)
                if rank == 0:
                    subs[wl] = rec
            if rank == 0:
                line["workloads"] = subs
        if rank == 0:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
