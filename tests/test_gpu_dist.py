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


# ---- the NVLink mailbox transport across real processes (split form) --------
# P2PTransport maps every peer's mailbox through CUDA IPC.  Here 2-3 processes
# share this box's one GPU, so the exchange runs in its split form: every rank
# publishes (device stores into the peers' IPC-mapped mailboxes, fence, epoch
# flags), the host barrier orders all publishes before any collect, and the
# collect then folds without waiting -- no kernel ever waits on another
# process's kernel.  This checks the IPC handle exchange and mapping, the
# cross-process stores and flags, epoch parity over several rounds, and the
# fold, against tf_combine and the one-GPU reduction.  Only the NVLink hop
# itself (a peer on another GPU) is left to a multi-GPU box.


def _xgpu_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1401_6235_b200 import dist as D
        from paper_1401_6235_b200 import reduce as R

        T = D.P2PTransport()
        out = []
        # (1) combine of given partials, 4 epochs (both parity buffers twice)
        for ep, dt in enumerate((torch.float64, torch.float32, torch.float64, torch.float32)):
            rng = np.random.default_rng(1000 + 10 * ep + rank)
            v = rng.uniform(-1, 1, 2) * np.array([1.0, 2.0**-40])
            part = torch.tensor(v, dtype=dt, device="cuda")
            counts = [0 if (ep == 2 and r == world - 1) else 5 for r in range(world)]
            mine = part.clone()
            T.publish(part, counts)
            torch.cuda.synchronize()
            dist.barrier()
            T.collect(part)
            torch.cuda.synchronize()
            allp = D.gather_partials(mine)  # gloo: host-side reference inputs
            ref = R.combine(allp, counts)
            out.append(("combine", ep, tuple(part.cpu().tolist()), (ref.value, ref.error)))
            dist.barrier()
        # (2) fused reduce + publish, then collect: every rop, f64 and f32
        rng = np.random.default_rng(77)
        x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-25, 26, n))
        y = rng.uniform(-1, 1, n)
        for rop in ("sum", "sum2", "dot"):
            for dt, npdt in ((torch.float64, np.float64), (torch.float32, np.float32)):
                L = R.tile_elems(npdt)
                lo, hi = D.shard_tiles(n, world, rank, L)
                local = [torch.from_numpy(x[lo:hi].astype(npdt)).cuda()]
                if rop != "sum":
                    local.append(torch.from_numpy(y[lo:hi].astype(npdt)).cuda())
                o = T.reduce(rop, local, D.shard_counts(n, world, L), publish_only=True)
                torch.cuda.synchronize()
                dist.barrier()
                T.collect(o)
                torch.cuda.synchronize()
                out.append(("reduce", rop, str(dt), tuple(o.cpu().tolist())))
                dist.barrier()
        out.append(("status", T.status()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_transport_ipc_across_processes_split_form(world):
    from paper_1401_6235_b200 import reduce as R

    n = 9 * 131072 + 777  # f32 tiles are 2x the f64 tile: ragged shards both ways
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_xgpu_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(77)
    x = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-25, 26, n))
    y = rng.uniform(-1, 1, n)
    whole = {}
    for dt, npdt in ((torch.float64, np.float64), (torch.float32, np.float32)):
        X = torch.from_numpy(x.astype(npdt)).cuda()
        Y = torch.from_numpy(y.astype(npdt)).cuda()
        whole[("sum", str(dt))] = R.vtsum(X)
        whole[("sum2", str(dt))] = R.vtsum2((X, Y))
        whole[("dot", str(dt))] = R.vtdot(X, Y)
    first = None
    for rank in range(world):
        items = res[rank]
        assert items[-1] == ("status", 0)
        for it in items[:-1]:
            if it[0] == "combine":
                _, ep, got, want = it
                assert got == want, (rank, ep)
            else:
                _, rop, dt, got = it
                w = whole[(rop, dt)]
                assert got == (w.value, w.error), (rank, rop, dt)
        if first is None:
            first = items
        assert items == first  # every rank ends with the same bits
