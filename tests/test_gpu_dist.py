"""The sharded reduction with the REAL device kernels across 2 and 3 ranks.

The ranks share the one GPU of this box and exchange partials over gloo (host
side), so no kernel waits on another rank (safe on a single GPU); each rank
reduces its tile-aligned shard with tf_reduce and folds the gathered partials
with tf_combine.  Every rank must get the one-GPU result bit for bit.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, rop, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1401_6235_b200 import dist as D
        from paper_1401_6235_b200 import reduce as R

        rng = np.random.default_rng(77)
        x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-25, 26, n))
        y = rng.uniform(-1, 1, n)
        L = R.tile_elems(np.float64)
        lo, hi = D.shard_tiles(n, world, rank, L)
        local = [torch.from_numpy(x[lo:hi].copy()).cuda()]
        if rop != "sum":
            local.append(torch.from_numpy(y[lo:hi].copy()).cuda())
        z = D.sharded_reduce(rop, local, n)
        q.put((rank, z.value, z.error))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("rop", ["sum", "dot"])
def test_sharded_reduce_device_kernels(world, rop):
    from paper_1401_6235_b200 import reduce as R

    n = 11 * 65536 + 4321
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, rop, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(77)
    x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-25, 26, n))
    y = rng.uniform(-1, 1, n)
    X = torch.from_numpy(x).cuda()
    whole = R.vtsum(X) if rop == "sum" else R.vtdot(X, torch.from_numpy(y).cuda())
    for _, z0, z1 in res:
        assert (z0, z1) == (whole.value, whole.error)
