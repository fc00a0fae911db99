"""Multi-GPU sharding: one process per GPU (torch.distributed over NCCL).

Elementwise kernels and Horner shard into independent contiguous slices with no
communication at all.  Reductions have one real exchange step: every rank
reduces its shard to a 16-byte twofold partial, the partials are all-gathered
(NCCL over NVLink/NVSwitch), and every rank folds them with the same
adjacent-pair ``_tadd`` tree (``tf_combine``).  NCCL's own sum is never used:
it drops z1 and its order depends on topology.

Shards for reductions are blocks of B = 2^ceil(log2(ceil(T/G))) whole tiles
(T tiles of L elements, G ranks), so each shard is a complete subtree of the
canonical tree: the result is bit-identical for every G and to the one-GPU
result ("Canonical reduction order").
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence, Tuple

try:
    import torch
    import torch.distributed as dist
except Exception:  # pragma: no cover
    torch = None
    dist = None


def shard_elementwise(n: int, world: int, rank: int, align: int = 2) -> Tuple[int, int]:
    """Contiguous [lo, hi) slice of n elements for `rank`, cut at multiples of
    `align` elements (16-byte boundaries keep every shard on the vector path)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-n // world)
    per = -(-per // align) * align
    lo = min(rank * per, n)
    hi = min(lo + per, n)
    return lo, hi


def shard_tiles(n: int, world: int, rank: int, tile: int) -> Tuple[int, int]:
    """Element range [lo, hi) of `rank`'s reduction shard: an aligned
    power-of-two block of whole tiles (a complete subtree of the tile tree)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    T = -(-n // tile)
    per = -(-T // world) if T else 0
    B = 1
    while B < per:
        B <<= 1
    t0 = min(rank * B, T)
    t1 = min(t0 + B, T)
    return min(t0 * tile, n), min(t1 * tile, n)


def shard_counts(n: int, world: int, tile: int) -> list:
    return [hi - lo for lo, hi in (shard_tiles(n, world, r, tile) for r in range(world))]


def gather_partials(partial, group=None):
    """All-gather each rank's partial (2 elements, or any small shape, e.g. the
    (2, 2) dot and sum partials of one step) into a (world, *shape) tensor in
    rank order — ONE collective however many reductions it carries."""
    world = dist.get_world_size(group)
    shape = tuple(partial.shape)
    out = torch.empty((world,) + shape, dtype=partial.dtype, device=partial.device)
    src = partial.contiguous()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out.reshape(world, -1), src.reshape(-1), group=group)
    else:  # gloo (CPU tests, single-GPU dry runs): gather through host tensors
        host = src.cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        for r in range(world):
            out[r] = parts[r].to(out.device)
    return out


def sharded_reduce(rop: str, local: Sequence, n: int, group=None,
                   reduce_fn: Optional[Callable] = None,
                   combine_fn: Optional[Callable] = None, tile: Optional[int] = None,
                   transport=None):
    """Reduce a globally sharded plane set; every rank returns the same Twofold.

    ``local`` holds this rank's planes (its shard_tiles slice).  reduce_fn /
    combine_fn default to the device kernels; tests on CPU (gloo) inject others.
    """
    from . import reduce as R

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if tile is None:
        import numpy as np

        dt = np.float64 if local[0].dtype == torch.float64 else np.float32
        tile = R.tile_elems(dt)
    lo, hi = shard_tiles(n, world, rank, tile)
    if local[0].shape[0] != hi - lo:
        raise ValueError("sharded_reduce: rank %d holds %d elements, its shard is %d"
                         % (rank, local[0].shape[0], hi - lo))
    if transport is not None and reduce_fn is None:
        # NVLink peer-memory path: local reduction and exchange in ONE launch
        counts = shard_counts(n, world, tile)
        v = transport.reduce(rop, local, counts).cpu().tolist()
        return R.Twofold(v[0], v[1])
    if reduce_fn is None:
        fn = {"sum": R.vtsum, "sum2": lambda a, b, out: R.vtsum2((a, b), out=out),
              "dot": R.vtdot}[rop]
        part = torch.empty(2, dtype=local[0].dtype, device=local[0].device)
        if hi > lo:
            fn(*local, out=part)
        else:
            part.zero_()
    else:
        part = reduce_fn(rop, local)
    if transport is not None:  # NVLink peer-memory combine (P2PTransport), no NCCL
        counts = shard_counts(n, world, tile)
        transport.combine(part, counts)
        v = part.cpu().tolist()
        return R.Twofold(v[0], v[1])
    allp = gather_partials(part, group)
    counts = shard_counts(n, world, tile)
    if combine_fn is None:
        return R.combine(allp, counts)
    return combine_fn(allp, counts)


__all__ = ["shard_elementwise", "shard_tiles", "shard_counts", "gather_partials",
           "sharded_reduce", "P2PTransport"]


class P2PTransport:
    """Cross-GPU combine over NVLink peer memory, without NCCL (opt-in).

    Every rank maps every other rank's mailbox through CUDA IPC; after the
    local reduction one device thread stores the 16-byte partial into all
    peers' mailboxes, waits for all of theirs and folds them with the same
    adjacent-pair tree as ``tf_combine`` (csrc/xgpu.cu), so results are
    bit-identical to the NCCL path.  Collective: every rank constructs it and
    calls ``combine`` the same number of times.  With no process group (or a
    world of 1) it runs single-rank, which is how it is tested on one GPU.
    """

    def __init__(self, group=None, device=None):
        import ctypes

        from . import _lib

        self._lib = _lib
        self.dev = torch.cuda.current_device() if device is None else device
        _lib.ensure_device(self.dev)
        use_dist = dist is not None and dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if use_dist else 1
        self.rank = dist.get_rank(group) if use_dist else 0
        h = (ctypes.c_char * 64)()
        _lib.check(_lib.lib().tf_xgpu_mailbox(self.dev, h), "P2PTransport")
        handles = [bytes(h)]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(h), group=group)
        blob = b"".join(handles)
        _lib.check(_lib.lib().tf_xgpu_open(self.dev, self.world, self.rank, blob), "P2PTransport")

    def combine(self, partial, counts):
        """partial: this rank's 2-element CUDA tensor (overwritten with the result)."""
        import ctypes

        dt = self._lib.TF_F64 if partial.dtype == torch.float64 else self._lib.TF_F32
        c = (ctypes.c_int64 * self.world)(*[int(v) for v in counts])
        with torch.cuda.device(partial.device):
            s = torch.cuda.current_stream(partial.device).cuda_stream
            rc = self._lib.lib().tf_xgpu_combine(dt, partial.data_ptr(), c, s)
        self._lib.check(rc, "P2PTransport.combine")
        return partial

    def publish(self, partial, counts):
        """Split form, phase 1 (tf_xgpu_publish): store this rank's partial in every
        peer's mailbox and return.  ``collect`` must follow on every rank once all
        ranks' publishes have completed (stream sync + host barrier)."""
        import ctypes

        dt = self._lib.TF_F64 if partial.dtype == torch.float64 else self._lib.TF_F32
        c = (ctypes.c_int64 * self.world)(*[int(v) for v in counts])
        with torch.cuda.device(partial.device):
            s = torch.cuda.current_stream(partial.device).cuda_stream
            rc = self._lib.lib().tf_xgpu_publish(dt, partial.data_ptr(), c, s)
        self._lib.check(rc, "P2PTransport.publish")
        return partial

    def collect(self, out):
        """Split form, phase 2 (tf_xgpu_collect): fold the published partials into
        ``out`` (2-element CUDA tensor of the published dtype)."""
        dt = self._lib.TF_F64 if out.dtype == torch.float64 else self._lib.TF_F32
        with torch.cuda.device(out.device):
            s = torch.cuda.current_stream(out.device).cuda_stream
            rc = self._lib.lib().tf_xgpu_collect(dt, out.data_ptr(), s)
        self._lib.check(rc, "P2PTransport.collect")
        return out

    def reduce(self, rop, planes, counts, out=None, publish_only=False):
        """This rank's reduction of ``planes`` (its shard, CUDA tensors) fused with
        the exchange: ONE launch (tf_xgpu_reduce) leaves the global twofold in
        ``out`` (a 2-element CUDA tensor; allocated if None) on the current stream.
        ``publish_only``: the split form (tf_xgpu_reduce_publish) — ``out`` gets the
        local result, published to the peers; ``collect(out)`` finishes it."""
        import ctypes

        from . import reduce as R
        from .kernels import _describe, _dtype_id

        who = "P2PTransport.reduce"
        ps = [_describe(who, p) for p in planes]
        first = ps[0]
        if any(p.kind != "cuda" for p in ps):
            raise ValueError("P2PTransport.reduce: planes must be CUDA tensors")
        if any(p.n != first.n or p.dtype != first.dtype for p in ps):
            raise ValueError("P2PTransport.reduce: planes differ in length or dtype")
        dt = _dtype_id(first.dtype)
        tdt = torch.float64 if dt == self._lib.TF_F64 else torch.float32
        if out is None:
            out = torch.empty(2, dtype=tdt, device="cuda:%d" % first.device)
        ws = R.workspace(first.device, dt, max(first.n, 1))
        c = (ctypes.c_int64 * self.world)(*[int(v) for v in counts])
        with torch.cuda.device(first.device):
            s = torch.cuda.current_stream(first.device).cuda_stream
            fn = self._lib.lib().tf_xgpu_reduce_publish if publish_only else \
                self._lib.lib().tf_xgpu_reduce
            rc = fn(self._lib.ROP_IDS[rop], dt, first.n, first.ptr,
                    ps[1].ptr if len(ps) > 1 else None, out.data_ptr(), ws.data_ptr(), ws.numel(),
                    c, s)
        self._lib.check(rc, who)
        return out

    def status(self):
        return self._lib.lib().tf_xgpu_status(self.dev)
