"""Multi-process (world_size 2 and 3) CPU tests of the sharded-reduction host
path over gloo: shard boundaries, the all-gather in rank order and the combine
tree.  The device kernels are swapped for the oracle (checker) here because
this container has no GPU; on a GPU box the same sharded_reduce drives
tf_reduce / NCCL / tf_combine (bench.py config4, tests/test_gpu_reduce.py)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

GEOM = (2, 8, 4)  # small tiles so a few thousand elements span many tiles
TILE = GEOM[0] * GEOM[1] * GEOM[2]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, rop, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as o
        from paper_1401_6235_b200 import dist as D

        rng = np.random.default_rng(1234)
        x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))
        y = rng.uniform(-1, 1, n)
        lo, hi = D.shard_tiles(n, world, rank, TILE)
        local = [torch.from_numpy(x[lo:hi].copy())]
        if rop != "sum":
            local.append(torch.from_numpy(y[lo:hi].copy()))

        def reduce_fn(rop_, planes):
            if planes[0].shape[0] == 0:
                return torch.zeros(2, dtype=torch.float64)
            a = planes[0].numpy()
            b = planes[1].numpy() if len(planes) > 1 else None
            z = o.reduce(rop_, a, b, geometry=GEOM, nthreads=1)
            return torch.tensor([float(z[0]), float(z[1])], dtype=torch.float64)

        def combine_fn(allp, counts):
            return o.combine(allp.numpy(), counts)

        z = D.sharded_reduce(rop, local, n, reduce_fn=reduce_fn, combine_fn=combine_fn,
                             tile=TILE)
        q.put((rank, float(z[0]), float(z[1])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("rop", ["sum", "dot", "sum2"])
def test_sharded_reduce_matches_single_shard(oracle, world, rop):
    n = 41 * TILE + 17
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, rop, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(1234)
    x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 31, n))
    y = rng.uniform(-1, 1, n)
    want = oracle.reduce(rop, x, None if rop == "sum" else y, geometry=GEOM)
    for _, z0, z1 in res:
        assert (z0, z1) == (float(want[0]), float(want[1]))


def test_shard_tiles_partition_properties():
    from paper_1401_6235_b200 import dist as D

    for n in (0, 1, TILE - 1, TILE, 5 * TILE + 3, 64 * TILE, 100 * TILE + 1):
        for G in (1, 2, 3, 4, 5, 8):
            ranges = [D.shard_tiles(n, G, r, TILE) for r in range(G)]
            # contiguous, covering, in rank order
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            # every non-final non-empty shard is a power-of-two block of whole tiles
            T = -(-n // TILE)
            for r, (lo, hi) in enumerate(ranges):
                if hi > lo:
                    assert lo % TILE == 0
                    tiles = -(-(hi - lo) // TILE)
                    B = tiles if hi < n else None
                    if B is not None:
                        assert B & (B - 1) == 0
            # empty shards form a suffix
            empties = [hi == lo for lo, hi in ranges]
            if True in empties:
                k = empties.index(True)
                assert all(empties[k:]) or n == 0
            del T


def test_shard_elementwise_alignment():
    from paper_1401_6235_b200 import dist as D

    for n in (0, 1, 7, 1000, 2**20 + 3):
        for G in (1, 2, 4, 8):
            rs = [D.shard_elementwise(n, G, r) for r in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for lo, hi in rs:
                assert lo % 2 == 0 or lo == n
