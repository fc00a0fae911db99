"""GPU parity of the elementwise kernels (run on a B200 via gpurun / the driver).

Every comparison is bit-exact on both planes, NaN positions compared by isnan
(x86 and NVIDIA NaN payloads differ; test_kernels.py:148-155 compares NaN the
same way).  Sources of truth: the reference-generated goldens and the oracle.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import GOLDEN  # noqa: E402

pytestmark = pytest.mark.gpu

ELEM = np.load(GOLDEN / "elementwise.npz")
NAMES = sorted({k.split("/")[0] for k in ELEM.files})
DEV = "cuda:0"


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return np.array_equal(a[~na].view(u), b[~nb].view(u))


def first_mismatch(a, b):
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    bad = np.flatnonzero((a.view(u) != b.view(u)) & ~(np.isnan(a) & np.isnan(b)))
    return bad[:5]


def run_device(name, ins, offset=0, offsets=None):
    """Run one op on the device over copies of the host planes; optional
    element offsets make the planes misaligned views."""
    from paper_1401_6235_b200 import kernels as K

    n = ins[0].shape[0]
    dt = torch.float64 if ins[0].dtype == np.float64 else torch.float32
    offs = offsets or [offset] * (len(ins) + 2)
    planes = []
    for k, p in enumerate(ins):
        buf = torch.empty(n + offs[k], dtype=dt, device=DEV)
        v = buf[offs[k]:]
        v.copy_(torch.from_numpy(np.ascontiguousarray(p)))
        planes.append(v)
    outs, bufs = [], []
    for k in range(2):
        o = offs[len(ins) + k]
        buf = torch.full((n + o + 8,), 7.0, dtype=dt, device=DEV)  # guards either side
        bufs.append((buf, o))
        outs.append(buf[o:o + n])
    if name in K.RAW_OPS:
        K.raw_loop(name)(*planes, *outs)
    else:
        spec = K.KERNELS[name]
        if spec.arity == "22":
            spec.func(K.TwofoldArray(planes[0], planes[1]), K.TwofoldArray(planes[2], planes[3]), K.TwofoldArray(*outs))
        elif spec.arity == "21":
            spec.func(K.TwofoldArray(planes[0], planes[1]), planes[2], K.TwofoldArray(*outs))
        elif spec.arity == "11":
            spec.func(planes[0], planes[1], K.TwofoldArray(*outs))
        elif spec.arity == "u2":
            spec.func(K.TwofoldArray(planes[0], planes[1]), K.TwofoldArray(*outs))
        else:
            spec.func(planes[0], K.TwofoldArray(*outs))
    torch.cuda.synchronize()
    for buf, o in bufs:  # nothing written outside the n output elements
        assert bool((buf[:o] == 7).all()) and bool((buf[o + n:] == 7).all()), (name, offs)
    return outs[0].cpu().numpy(), outs[1].cpu().numpy()


def golden_inputs(name, fmt):
    ins, k = [], 0
    while "%s/%s/in%d" % (name, fmt, k) in ELEM.files:
        ins.append(ELEM["%s/%s/in%d" % (name, fmt, k)])
        k += 1
    return ins


@pytest.mark.parametrize("fmt", ["f64", "f32"])
@pytest.mark.parametrize("name", NAMES)
def test_device_matches_reference_golden(name, fmt):
    ins = golden_inputs(name, fmt)
    r0, r1 = run_device(name, ins)
    w0, w1 = ELEM["%s/%s/out0" % (name, fmt)], ELEM["%s/%s/out1" % (name, fmt)]
    assert bits_equal(r0, w0), (name, first_mismatch(r0, w0))
    assert bits_equal(r1, w1), (name, first_mismatch(r1, w1))


@pytest.mark.parametrize("fmt", ["f64", "f32"])
@pytest.mark.parametrize("name", ["vtadd2", "vtdiv1", "vtsqrt1", "vtmul", "vtsqrt", "vpmul2"])
def test_device_misaligned_views(name, fmt):
    # common misalignment (scalar head + vector body + scalar tail) and mixed
    # misalignments (scalar grid-stride path) must give the same bits
    ins = golden_inputs(name, fmt)
    w0, w1 = ELEM["%s/%s/out0" % (name, fmt)], ELEM["%s/%s/out1" % (name, fmt)]
    for offset in (1, 3):
        r0, r1 = run_device(name, ins, offset=offset)
        assert bits_equal(r0, w0) and bits_equal(r1, w1), (name, offset)
    mixed = [k % 3 for k in range(len(ins) + 2)]
    r0, r1 = run_device(name, ins, offsets=mixed)
    assert bits_equal(r0, w0) and bits_equal(r1, w1), (name, "mixed")
    # equal modulo 16 bytes, different modulo 32 (still the all-scalar path, which
    # streams at the vector kernels' rate: profiles/r2s5_halfaligned_probe.txt)
    e16 = 2 if fmt == "f64" else 4
    for lead in (0, 1):
        half = [lead + e16 * (k % 4) for k in range(len(ins) + 2)]
        r0, r1 = run_device(name, ins, offsets=half)
        assert bits_equal(r0, w0) and bits_equal(r1, w1), (name, "half-aligned", lead)


def _config1(n, seed):
    # BASELINE config 1: x0,y0 ~ U[-1,1]; x1 = x0*2^-53*U[-1,1], likewise y1
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(-1, 1, n)
    x1 = x0 * 2.0**-53 * rng.uniform(-1, 1, n)
    y0 = rng.uniform(-1, 1, n)
    y1 = y0 * 2.0**-53 * rng.uniform(-1, 1, n)
    return x0, x1, y0, y1


@pytest.mark.parametrize("name", ["vtadd2", "vtmul2"])
def test_config1_bit_exact_vs_oracle(oracle, name):
    ins = _config1(2**20, 1 if name == "vtadd2" else 2)
    r0, r1 = run_device(name, ins)
    w0, w1 = oracle.elementwise(name, *ins)
    assert bits_equal(r0, w0) and bits_equal(r1, w1)


def _config2_inputs(name, n, seed):
    # BASELINE config 2 distributions (log-uniform heads, tails head*2^-53*U[-1,1])
    rng = np.random.default_rng(seed)

    def head(lo, hi, signed=True):
        v = np.exp2(rng.uniform(lo, hi, n))
        return v * rng.choice([-1.0, 1.0], n) if signed else v

    def tail(h):
        return h * 2.0**-53 * rng.uniform(-1, 1, n)

    if name == "vtsqrt1":
        x0 = head(-20, 20, signed=False)
        return x0, tail(x0)
    x0 = head(-20, 20)
    y0 = head(-10, 10, signed=False) if name == "vtdiv2" else head(-20, 20)
    return x0, tail(x0), y0, tail(y0)


@pytest.mark.parametrize("name", ["vtadd2", "vtsub2", "vtmul2", "vtdiv2", "vtsqrt1"])
def test_config2_ops_bit_exact_vs_oracle(oracle, name):
    n = (1 << 22) + 5
    ins = _config2_inputs(name, n, 20 + len(name))
    r0, r1 = run_device(name, ins)
    w0, w1 = oracle.elementwise(name, *ins)
    assert bits_equal(r0, w0), first_mismatch(r0, w0)
    assert bits_equal(r1, w1), first_mismatch(r1, w1)


@pytest.mark.parametrize("name", ["vtadd2", "vtmul2", "vtdiv2"])
def test_config3_f32_bit_exact_vs_oracle(oracle, name):
    n = (1 << 22) + 3
    rng = np.random.default_rng(33)
    x0 = rng.uniform(-1, 1, n).astype(np.float32)
    x1 = (x0 * np.float32(2.0**-24) * rng.uniform(-1, 1, n).astype(np.float32)).astype(np.float32)
    if name == "vtdiv2":
        y0 = rng.uniform(0.5, 2, n).astype(np.float32)
    else:
        y0 = rng.uniform(-1, 1, n).astype(np.float32)
    y1 = (y0 * np.float32(2.0**-24) * rng.uniform(-1, 1, n).astype(np.float32)).astype(np.float32)
    ins = (x0, x1, y0, y1)
    r0, r1 = run_device(name, ins)
    w0, w1 = oracle.elementwise(name, *ins)
    assert bits_equal(r0, w0) and bits_equal(r1, w1)


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_head_tail_boundary_sweep_vs_oracle(oracle, fmt):
    # every (head, tail) pair of the single-step kernels: the common misalignment sets the
    # scalar head (0 .. 32/sizeof(T) - 1 elements), n the tail; lengths around one vector,
    # one CTA (256 vectors of 16 or 32 bytes) and two CTAs.  Outputs are guard-banded by
    # run_device.  vtsqrt runs the 32-byte kernel, the others the 16-byte one.
    dtype = np.float64 if fmt == "f64" else np.float32
    e32 = 4 if fmt == "f64" else 8
    rng = np.random.default_rng(21)
    lengths = sorted(set(list(range(1, 3 * e32 + 2)) +
                         [256 * e32 // 2 + d for d in (-1, 0, 1)] +
                         [256 * e32 + d for d in range(-e32, e32 + 1)] +
                         [512 * e32 + d for d in (-1, 0, 1, e32 + 1)]))
    for name, nin in (("vtadd2", 4), ("vtdiv2", 4), ("vtsqrt1", 2), ("vtsqrt", 1)):
        for off in range(e32):
            for n in lengths:
                ins = [rng.uniform(0.5, 2, n).astype(dtype) for _ in range(nin)]
                w0, w1 = oracle.elementwise(name, *ins)
                r0, r1 = run_device(name, ins, offset=off)
                assert bits_equal(r0, w0) and bits_equal(r1, w1), (name, fmt, off, n)


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_all_ops_random_wide_vs_oracle(oracle, fmt):
    # every op at a size with many CTAs, wide exponents, subnormal-producing tails
    from paper_1401_6235_b200 import kernels as K

    dtype = np.float64 if fmt == "f64" else np.float32
    n = 300_001
    rng = np.random.default_rng(9)
    me = 300 if fmt == "f64" else 40
    for name in list(K.KERNELS) + ["div_rem", "sqrt_resid"]:
        nin = {4: 4, 3: 3, 2: 2, 1: 1}[{"22": 4, "21": 3, "11": 2, "u2": 2, "u1": 1}.get(
            K.KERNELS[name].arity if name in K.KERNELS else ("11" if name == "div_rem" else "u1"))]
        with np.errstate(all="ignore"):
            ins = []
            for k in range(nin):
                v = rng.uniform(1, 2, n) * np.exp2(rng.integers(-me, me, n)) * rng.choice([-1.0, 1.0], n)
                if name in ("vtsqrt1", "vtsqrt", "sqrt_resid") and k == 0:
                    v = np.abs(v)
                ins.append(v.astype(dtype))
        with np.errstate(all="ignore"):
            w0, w1 = oracle.elementwise(name, *ins)
        r0, r1 = run_device(name, ins)
        assert bits_equal(r0, w0), (name, first_mismatch(r0, w0))
        assert bits_equal(r1, w1), (name, first_mismatch(r1, w1))


def test_host_planes_path_matches_oracle(oracle):
    # numpy planes in and out: the reference's calling convention, staged through
    # the device by tf_elementwise_host (several pipeline chunks)
    from paper_1401_6235_b200 import kernels as K

    n = 5 * (1 << 21) + 17
    ins = _config2_inputs("vtdiv2", n, 4)
    out = K.empty_twofold(n, np.float64, device="cpu")
    K.vtdiv2(K.TwofoldArray(ins[0], ins[1]), K.TwofoldArray(ins[2], ins[3]), out)
    w0, w1 = oracle.elementwise("vtdiv2", *ins)
    assert bits_equal(out.value, w0) and bits_equal(out.error, w1)
    # pinned host planes take the same path
    outp = K.empty_twofold(n, np.float64, device="cpu", pin_memory=True)
    K.vtdiv2(K.TwofoldArray(ins[0], ins[1]), K.TwofoldArray(ins[2], ins[3]), outp)
    assert bits_equal(outp.value, w0) and bits_equal(outp.error, w1)


# ---- the reference's test_kernels.py contract, re-run on device planes ----

def _t(a):
    return torch.as_tensor(np.asarray(a), device=DEV)


def test_length_one_matches_reference_value():
    from paper_1401_6235_b200 import kernels as K

    x = K.TwofoldArray(_t([1.0]), _t([-(2.0**-53)]))
    y = K.TwofoldArray(_t([2.0**-53]), _t([-(2.0**-106)]))
    out = K.empty_twofold(1, torch.float64)
    K.vtadd2(x, y, out)
    # tadd((1,-2^-53),(2^-53,-2^-106)): TwoSum(1, 2^-53) = (1, 2^-53)
    assert (out.value.item(), out.error.item()) == (1.0, (-(2.0**-53) + -(2.0**-106)) + 2.0**-53)


def test_inputs_may_alias_each_other(oracle):
    from paper_1401_6235_b200 import kernels as K

    v = np.array([1.0, 2.0, 3.0])
    e = np.array([2.0**-54, 0.0, -(2.0**-53)])
    x = K.TwofoldArray(_t(v), _t(e))
    out = K.empty_twofold(3, torch.float64)
    K.vtadd2(x, x, out)
    w0, w1 = oracle.elementwise("vtadd2", v, e, v, e)
    assert bits_equal(out.value.cpu().numpy(), w0) and bits_equal(out.error.cpu().numpy(), w1)


def test_specials_flow_through_kernels():
    from paper_1401_6235_b200 import kernels as K

    out = K.empty_twofold(3, torch.float64, K.CoupledArray)
    K.vtdiv(_t([1.0, 0.0, -1.0]), _t([0.0, 0.0, np.inf]), out)
    v, e = out.value.cpu().numpy(), out.error.cpu().numpy()
    assert v[0] == np.inf and np.isnan(e[0])
    assert np.isnan(v[1]) and np.isnan(e[1])
    assert v[2] == 0.0 and np.signbit(v[2])
    out = K.empty_twofold(1, torch.float64, K.CoupledArray)
    K.vtsqrt(_t([-1.0]), out)
    assert np.isnan(out.value.item()) and np.isnan(out.error.item())


def test_dotted_kernel_outputs_are_coupled():
    from paper_1401_6235_b200 import kernels as K

    rng = np.random.default_rng(7)
    a = rng.uniform(1, 2, 1000) * np.exp2(rng.integers(-3, 4, 1000)) * rng.choice([-1.0, 1.0], 1000)
    b = rng.uniform(1, 2, 1000) * np.exp2(rng.integers(-3, 4, 1000)) * rng.choice([-1.0, 1.0], 1000)
    out = K.empty_twofold(1000, torch.float64, K.CoupledArray)
    for f in (K.vtadd, K.vtmul, K.vtdiv):
        f(_t(a), _t(b), out)
        v, e = out.value.cpu().numpy(), out.error.cpu().numpy()
        assert np.all(np.abs(e) <= np.spacing(np.abs(v)) / 2)


def test_empty_arrays_are_a_no_op():
    from paper_1401_6235_b200 import kernels as K

    x = K.TwofoldArray(torch.empty(0, dtype=torch.float64, device=DEV),
                       torch.empty(0, dtype=torch.float64, device=DEV))
    out = K.empty_twofold(0, torch.float64)
    K.vtadd2(x, x, out)
    assert out.value.shape == (0,)


def test_device_validation_before_launch():
    from paper_1401_6235_b200 import kernels as K

    x = K.TwofoldArray(_t(np.ones(8)), _t(np.ones(8)))
    out = K.TwofoldArray(torch.full((8,), 7.0, dtype=torch.float64, device=DEV),
                         torch.full((8,), 7.0, dtype=torch.float64, device=DEV))
    with pytest.raises(ValueError, match="alias"):
        K.vtadd2(x, x, K.TwofoldArray(x.value, out.error))
    with pytest.raises(ValueError, match="overlap"):
        K.vtadd2(x, x, K.TwofoldArray(out.value, out.value))
    with pytest.raises(ValueError, match="mix"):
        K.vtadd2(x, K.TwofoldArray(np.ones(8), np.ones(8)), out)
    with pytest.raises(ValueError, match="lengths differ"):
        K.vtadd2(x, K.TwofoldArray(x.value[:4], x.error[:4]), out)
    torch.cuda.synchronize()
    assert torch.all(out.value == 7.0) and torch.all(out.error == 7.0)


def test_selftest_and_dotted_baselines():
    from paper_1401_6235_b200 import _lib

    assert _lib.lib().tf_selftest(0) == 0
    n = 1001
    rng = np.random.default_rng(1)
    x = _t(rng.uniform(1, 2, n))
    y = _t(rng.uniform(1, 2, n))
    r = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    for base, ref in ((0, x + y), (1, x * y), (2, x / y), (3, torch.sqrt(x)), (4, x)):
        assert _lib.lib().tf_dotted(base, 1, n, x.data_ptr(), y.data_ptr(), r.data_ptr(), s) == 0
        torch.cuda.synchronize()
        assert torch.equal(r, ref), base


def test_host_batch_matches_oracle_and_rejects_chains(oracle):
    # several ops on host planes in one pipelined pass: shared inputs cross the
    # link once, every op's outputs come back, results equal one-by-one calls
    from paper_1401_6235_b200 import kernels as K

    n = 3 * (1 << 21) + 11
    a = _config2_inputs("vtadd2", n, 71)
    d = _config2_inputs("vtdiv2", n, 72)
    q = _config2_inputs("vtsqrt1", n, 73)
    X, Y = K.TwofoldArray(a[0], a[1]), K.TwofoldArray(a[2], a[3])
    outs = [K.empty_twofold(n, np.float64, device="cpu") for _ in range(4)]
    pinned = K.empty_twofold(n, np.float64, device="cpu", pin_memory=True)
    K.host_batch([("vtadd2", X, Y, outs[0]), ("vtmul2", X, Y, outs[1]),
                  ("vtdiv2", X, K.TwofoldArray(d[2], d[3]), outs[2]),
                  ("vtsqrt1", K.TwofoldArray(q[0], q[1]), outs[3]),
                  ("vtsub2", X, Y, pinned)])
    for o, (name, ins) in zip(outs + [pinned], [("vtadd2", a), ("vtmul2", a),
                                                ("vtdiv2", (a[0], a[1], d[2], d[3])),
                                                ("vtsqrt1", q), ("vtsub2", a)]):
        w0, w1 = oracle.elementwise(name, *ins)
        assert bits_equal(o.value, w0) and bits_equal(o.error, w1), name
    with pytest.raises(ValueError, match="alias"):
        K.host_batch([("vtadd2", X, Y, outs[0]), ("vtmul2", outs[0], Y, outs[1])])


def test_host_batch_of_64_ops_uses_short_chunks(oracle):
    # 64 ops = 132 staged planes: the pipeline shortens its chunks to stay in the
    # staging budget (several chunks per plane here) — bits must not change
    from paper_1401_6235_b200 import kernels as K

    n = (1 << 20) + 3
    a = _config2_inputs("vtadd2", n, 81)
    X, Y = K.TwofoldArray(a[0], a[1]), K.TwofoldArray(a[2], a[3])
    names = ["vtadd2", "vtsub2", "vtmul2", "vtdiv2", "vpadd2", "vpsub2", "vpmul2", "vpdiv2"]
    calls, outs = [], []
    for k in range(64):
        o = K.empty_twofold(n, np.float64, device="cpu")
        outs.append(o)
        calls.append((names[k % len(names)], X, Y, o))
    K.host_batch(calls)
    want = {name: oracle.elementwise(name, *a) for name in names}
    for k, o in enumerate(outs):
        w0, w1 = want[names[k % len(names)]]
        assert bits_equal(o.value, w0) and bits_equal(o.error, w1), k


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_all_ops_on_random_bit_patterns(oracle, fmt):
    # every IEEE class (subnormals, infinities, NaNs, signed zeros, huge/tiny
    # magnitudes) drawn from raw bit patterns: device == oracle, NaN by position
    from paper_1401_6235_b200 import kernels as K

    dtype = np.float64 if fmt == "f64" else np.float32
    u = np.uint64 if fmt == "f64" else np.uint32
    rng = np.random.default_rng(31337)
    n = 200_003
    for name in list(K.KERNELS) + ["div_rem", "sqrt_resid"]:
        nin = oracle.NUM_INPUTS[name]
        ins = []
        for _ in range(nin):
            raw = rng.integers(0, np.iinfo(u).max, n, dtype=u, endpoint=True).view(dtype)
            ordinary = (rng.uniform(-4, 4, n) * np.exp2(rng.integers(-40, 40, n))).astype(dtype)
            ins.append(np.where(rng.random(n) < 0.5, raw, ordinary).astype(dtype))
        with np.errstate(all="ignore"):
            w0, w1 = oracle.elementwise(name, *ins)
        r0, r1 = run_device(name, ins)
        assert bits_equal(r0, w0), (name, first_mismatch(r0, w0))
        assert bits_equal(r1, w1), (name, first_mismatch(r1, w1))


def test_cuda_graph_capture_and_replay(oracle):
    # the launchers are CUDA-graph safe: a captured step of several ops (and a
    # reduction) replays with the same bits as eager execution
    from paper_1401_6235_b200 import kernels as K
    from paper_1401_6235_b200 import reduce as R

    n = (1 << 20) + 3
    ins = _config2_inputs("vtdiv2", n, 91)
    X = K.TwofoldArray(_t(ins[0]), _t(ins[1]))
    Y = K.TwofoldArray(_t(ins[2]), _t(ins[3]))
    o1, o2 = K.empty_twofold(n, torch.float64), K.empty_twofold(n, torch.float64)
    red = torch.empty(2, dtype=torch.float64, device=DEV)
    o3, o4 = K.empty_twofold(n, torch.float64), K.empty_twofold(n, torch.float64)
    s = torch.cuda.Stream()

    pair = torch.empty((2, 2), dtype=torch.float64, device=DEV)

    def step():
        K.vtdiv2(X, Y, o1)
        K.vtadd2(o1, Y, o2)
        R.vtdot(o2.value, Y.value, out=red)
        K.batch([("vtdiv2", X, Y, o3), ("vtmul2", o2, Y, o4)])  # one launch
        R.batch([("vtdot", o2.value, Y.value), ("vtsum", o2.value)], out=pair)  # one pass

    with torch.cuda.stream(s):  # warm (self-test, occupancy, workspace) outside capture
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    for buf in (o1.value, o1.error, o2.value, o2.error, red, o3.value, o3.error,
                o4.value, o4.error, pair):
        buf.fill_(7.0)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    w1 = oracle.elementwise("vtdiv2", *ins)
    w2 = oracle.elementwise("vtadd2", w1[0], w1[1], ins[2], ins[3])
    assert bits_equal(o1.value.cpu().numpy(), w1[0]) and bits_equal(o1.error.cpu().numpy(), w1[1])
    assert bits_equal(o2.value.cpu().numpy(), w2[0]) and bits_equal(o2.error.cpu().numpy(), w2[1])
    wr = oracle.reduce("dot", w2[0], ins[2], geometry=R.geometry(np.float64))
    assert (red[0].item(), red[1].item()) == (float(wr[0]), float(wr[1]))
    ws = oracle.reduce("sum", w2[0], geometry=R.geometry(np.float64))
    assert pair.cpu().tolist() == [[float(wr[0]), float(wr[1])], [float(ws[0]), float(ws[1])]]
    w4 = oracle.elementwise("vtmul2", w2[0], w2[1], ins[2], ins[3])
    assert bits_equal(o3.value.cpu().numpy(), w1[0]) and bits_equal(o3.error.cpu().numpy(), w1[1])
    assert bits_equal(o4.value.cpu().numpy(), w4[0]) and bits_equal(o4.error.cpu().numpy(), w4[1])


def test_reused_pageable_planes_get_page_locked(oracle):
    # second use of a large pageable numpy plane registers it (DMA in place);
    # results stay bit-exact and the registration is released with the array
    import gc

    from paper_1401_6235_b200 import kernels as K

    n = 5 << 20  # 40 MiB per f64 plane
    ins = _config2_inputs("vtmul2", n, 5)
    x = K.TwofoldArray(ins[0].copy(), ins[1].copy())
    y = K.TwofoldArray(ins[2].copy(), ins[3].copy())
    out = K.empty_twofold(n, np.float64, device="cpu")
    w0, w1 = oracle.elementwise("vtmul2", *ins)
    for _ in range(K._REG_AFTER + 1):
        out.value[:] = 7.0
        K.vtmul2(x, y, out)
        assert bits_equal(out.value, w0) and bits_equal(out.error, w1)
    addrs = {a.ctypes.data for a in (x.value, x.error, y.value, y.error)}
    assert addrs <= set(K._REG), "reused planes were not page-locked"
    del x, y, out
    gc.collect()
    assert not (addrs & set(K._REG)), "registrations outlived their arrays"


# ---- device batch (tf_elementwise_batch): several ops in ONE launch ---------


def _batch_call(K, name, planes, out):
    spec = K.KERNELS[name]
    T = K.TwofoldArray
    if spec.arity == "22":
        return (name, T(planes[0], planes[1]), T(planes[2], planes[3]), out)
    if spec.arity == "21":
        return (name, T(planes[0], planes[1]), planes[2], out)
    if spec.arity == "11":
        return (name, planes[0], planes[1], out)
    if spec.arity == "u2":
        return (name, T(planes[0], planes[1]), out)
    return (name, planes[0], out)


@pytest.mark.parametrize("fmt", ["f64", "f32"])
@pytest.mark.parametrize("offset", [0, 1, "mixed"])
def test_device_batch_all_ops_match_one_by_one(fmt, offset):
    # every registry op in batches of 8 (plus a partial group), planes shared
    # between ops, wide exponents and specials; aligned, commonly misaligned and
    # mixed-misaligned (scalar path) views: bits equal to one launch per op
    from paper_1401_6235_b200 import kernels as K

    dt = torch.float64 if fmt == "f64" else torch.float32
    npdt = np.float64 if fmt == "f64" else np.float32
    n = 3 * 4096 + 29
    rng = np.random.default_rng(5)
    shared = []
    for k in range(4):
        v = (rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))).astype(npdt)
        v[:8] = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-310, 3.0, -2.5], dtype=npdt)
        shared.append(v)
    if offset == "mixed":
        offs = [1, 0, 3, 2]
    else:
        offs = [offset] * 4

    def plane(k):
        buf = torch.empty(n + offs[k], dtype=dt, device=DEV)
        p = buf[offs[k]:]
        p.copy_(torch.from_numpy(shared[k]))
        return p

    planes = [plane(k) for k in range(4)]
    names = [row[0] for row in K._TABLE]
    calls, outs, want = [], [], []
    for i, name in enumerate(names):
        nin = {"22": 4, "21": 3, "11": 2, "u2": 2, "u1": 1}[K.KERNELS[name].arity]
        ps = [planes[(i + k) % 4] for k in range(nin)]
        oo = offs[i % 4] if offset == "mixed" else offs[0]
        o = K.TwofoldArray(*(torch.full((n + oo,), 7.0, dtype=dt, device=DEV)[oo:]
                             for _ in range(2)))
        calls.append(_batch_call(K, name, ps, o))
        outs.append(o)
        w = K.empty_twofold(n, dt, device=DEV)
        K.KERNELS[name].func(*calls[-1][1:-1], w)
        want.append(w)
    K.batch(calls)
    torch.cuda.synchronize()
    for name, o, w in zip(names, outs, want):
        assert bits_equal(o.value.cpu().numpy(), w.value.cpu().numpy()), name
        assert bits_equal(o.error.cpu().numpy(), w.error.cpu().numpy()), name


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_device_batch_head_tail_boundary_sweep(oracle, fmt):
    # the batch kernels' head/tail CTA: every common misalignment x lengths around one
    # vector and one CTA, three ops over shared planes, guard bands around every output
    from paper_1401_6235_b200 import kernels as K

    dt = torch.float64 if fmt == "f64" else torch.float32
    npdt = np.float64 if fmt == "f64" else np.float32
    e32 = 4 if fmt == "f64" else 8
    rng = np.random.default_rng(33)
    lengths = sorted(set(list(range(1, 2 * e32 + 2)) + [256 * e32 // 2 + d for d in (-1, 0, 1)] +
                         [256 * e32 + d for d in (-e32, -1, 0, 1, e32)] + [512 * e32 + 3]))
    for off in range(e32):
        for n in lengths:
            ins = [rng.uniform(0.5, 2, n).astype(npdt) for _ in range(4)]

            def put(a):
                buf = torch.empty(n + off, dtype=dt, device=DEV)
                buf[off:].copy_(torch.from_numpy(a))
                return buf[off:]

            P = [put(a) for a in ins]
            X, Y = K.TwofoldArray(P[0], P[1]), K.TwofoldArray(P[2], P[3])
            bufs = [torch.full((n + off + 8,), 7.0, dtype=dt, device=DEV) for _ in range(6)]
            outs = [K.TwofoldArray(bufs[2 * i][off:off + n], bufs[2 * i + 1][off:off + n])
                    for i in range(3)]
            K.batch([("vtadd2", X, Y, outs[0]), ("vtdiv2", X, Y, outs[1]), ("vtsqrt1", X, outs[2])])
            torch.cuda.synchronize()
            for b in bufs:
                assert bool((b[:off] == 7).all()) and bool((b[off + n:] == 7).all()), (fmt, off, n)
            for name, o, w in (("vtadd2", outs[0], oracle.elementwise("vtadd2", *ins)),
                               ("vtdiv2", outs[1], oracle.elementwise("vtdiv2", *ins)),
                               ("vtsqrt1", outs[2], oracle.elementwise("vtsqrt1", ins[0], ins[1]))):
                assert bits_equal(o.value.cpu().numpy(), w[0]), (name, fmt, off, n)
                assert bits_equal(o.error.cpu().numpy(), w[1]), (name, fmt, off, n)


def test_device_batch_config2_step_vs_oracle(oracle):
    # the bench's config-2 step as one launch: x, y shared by add/sub/mul; the
    # divisor and sqrt planes of their own
    from paper_1401_6235_b200 import kernels as K

    n = (1 << 22) + 5
    a = _config2_inputs("vtadd2", n, 91)
    d = _config2_inputs("vtdiv2", n, 92)
    q = _config2_inputs("vtsqrt1", n, 93)
    t = lambda v: torch.from_numpy(v).to(DEV)  # noqa: E731
    X, Y = K.TwofoldArray(t(a[0]), t(a[1])), K.TwofoldArray(t(a[2]), t(a[3]))
    D = K.TwofoldArray(t(d[2]), t(d[3]))
    Q = K.TwofoldArray(t(q[0]), t(q[1]))
    outs = [K.empty_twofold(n, torch.float64, device=DEV) for _ in range(5)]
    K.batch([("vtadd2", X, Y, outs[0]), ("vtsub2", X, Y, outs[1]), ("vtmul2", X, Y, outs[2]),
             ("vtdiv2", X, D, outs[3]), ("vtsqrt1", Q, outs[4])])
    torch.cuda.synchronize()
    for o, (name, ins) in zip(outs, [("vtadd2", a), ("vtsub2", a), ("vtmul2", a),
                                     ("vtdiv2", (a[0], a[1], d[2], d[3])), ("vtsqrt1", q)]):
        w0, w1 = oracle.elementwise(name, *ins)
        assert bits_equal(o.value.cpu().numpy(), w0), name
        assert bits_equal(o.error.cpu().numpy(), w1), name


def test_device_batch_contract():
    # chains rejected before any launch (outputs untouched); n == 0 no-op; mixed
    # dtypes rejected; host planes route to host_batch
    from paper_1401_6235_b200 import _lib
    from paper_1401_6235_b200 import kernels as K

    n = 1000
    x = K.TwofoldArray(torch.ones(n, dtype=torch.float64, device=DEV),
                       torch.zeros(n, dtype=torch.float64, device=DEV))
    o1 = K.TwofoldArray(torch.full((n,), 5.0, dtype=torch.float64, device=DEV),
                        torch.full((n,), 5.0, dtype=torch.float64, device=DEV))
    o2 = K.empty_twofold(n, torch.float64, device=DEV)
    with pytest.raises(ValueError, match="alias"):
        K.batch([("vtadd2", x, x, o1), ("vtmul2", o1, x, o2)])
    torch.cuda.synchronize()
    assert (o1.value == 5.0).all() and (o1.error == 5.0).all()
    with pytest.raises(ValueError, match="mix"):
        K.batch([("vtadd2", x, x, o1), ("vtadd2", K.TwofoldArray(x.value.float(), x.error.float()),
                                        K.TwofoldArray(x.value.float(), x.error.float()),
                                        K.empty_twofold(n, torch.float32, device=DEV))])
    # outputs of different calls: identical planes are fine (later calls win, as
    # one by one); partially overlapping ones are rejected before any launch
    buf = torch.zeros(2 * n + 8, dtype=torch.float64, device=DEV)
    oa = K.TwofoldArray(buf[:n], buf[n + 8:])
    ob = K.TwofoldArray(buf[3:n + 3], torch.empty(n, dtype=torch.float64, device=DEV))
    with pytest.raises(ValueError, match="overlap"):
        K.batch([("vtadd2", x, x, oa), ("vtmul2", x, x, ob)])
    K.batch([("vtadd2", x, x, o2), ("vtmul2", x, x, o2)])  # same planes: vtmul2 wins
    w = K.empty_twofold(n, torch.float64, device=DEV)
    K.vtmul2(x, x, w)
    assert torch.equal(o2.value, w.value) and torch.equal(o2.error, w.error)
    hb = np.zeros(2 * n + 8)
    with pytest.raises(ValueError, match="overlap"):
        xh2 = K.TwofoldArray(np.ones(n), np.zeros(n))
        K.host_batch([("vtadd2", xh2, xh2, K.TwofoldArray(hb[:n], hb[n + 8:])),
                      ("vtmul2", xh2, xh2, K.TwofoldArray(hb[3:n + 3], np.empty(n)))])
    e = K.empty_twofold(0, torch.float64, device=DEV)
    z = K.TwofoldArray(x.value[:0], x.error[:0])
    K.batch([("vtadd2", z, z, e)])
    K.batch([])
    # the C ABI rejects more than 8 ops and unknown op ids
    ops = (__import__("ctypes").c_int * 9)(*([0] * 9))
    assert _lib.lib().tf_elementwise_batch(9, ops, _lib.TF_F64, 1, None, None, None) != 0
    # host planes: routed to the pipelined host path
    xh = K.TwofoldArray(np.ones(n), np.zeros(n))
    oh = K.empty_twofold(n, np.float64, device="cpu")
    K.batch([("vtadd2", xh, xh, oh)])
    assert (oh.value == 2.0).all() and (oh.error == 0.0).all()
