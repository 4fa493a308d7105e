"""Bandwidth-centric partitioner and its collectives (PAPER §6.1).

Mirrors the SPEC operations ``partition / allgather / reduce_scatter /
broadcast_fetch`` over the B200 tier store:

* ``partition`` shards a 1-D tensor with ceil(n/N) elements per rank and a
  zero-padded final shard, stored under ``key/rank<r>``.
* ``allgather`` rebuilds the full tensor on the GPU from every rank's shard
  in one libzinf gather (SM kernel or copy engines); shards may sit in HBM,
  pinned host DRAM (read over PCIe by the copy engine — the "cg" transfer)
  or NVMe.
* ``reduce_scatter`` folds per-rank contributions in fixed rank order
   with ``zi_reduce_scatter`` — fp32 accumulation for half
  inputs, bit-exact with the oracle.

``comm=None`` (or a LocalComm) is the SPEC's simulated-rank model: this
process holds every shard. With a DistComm each process holds its own
shard and the peers' shards are reached over NVLink (NCCL all-gather or
IPC-mapped P2P reads).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib, kernels
from .store import TierKind, TierStore, _as_tensor

_DT = {torch.float32: _lib.DT_F32, torch.float16: _lib.DT_F16, torch.float64: _lib.DT_F64,
       torch.bfloat16: _lib.DT_BF16}
_auto_key = itertools.count()
# barrier channel of the SPEC collectives over a DistComm (the GPT engine uses 0-2)
PARTITION_CHANNEL = 3


def shard_len(full_len: int, world_size: int) -> int:
    """ceil(full_len / world_size)."""
    if full_len < 1 or world_size < 1:
        raise ValueError("need full_len >= 1 and world_size >= 1")
    return -(-full_len // world_size)


def shard_key(key: str, rank: int) -> str:
    return f"{key}/rank{rank}"


@dataclass(frozen=True)
class PartitionedTensor:
    """A named 1-D tensor sharded across ranks."""
    key: str
    full_len: int
    dtype: torch.dtype
    world_size: int
    tier: TierKind

    @property
    def shard_len(self) -> int:
        return shard_len(self.full_len, self.world_size)

    def shard_key(self, rank: int) -> str:
        return shard_key(self.key, rank)

    def shard_range(self, rank: int) -> tuple[int, int]:
        L = self.shard_len
        s = min(rank * L, self.full_len)
        return s, min(s + L, self.full_len)


def _ranks(world_size: int, comm) -> range | list:
    if comm is None or comm.is_local:
        return range(world_size)
    if comm.world != world_size:
        raise ValueError("world_size disagrees with the communicator")
    return [comm.rank]


def make_shard(full: torch.Tensor, world_size: int, rank: int) -> torch.Tensor:
    """Rank's zero-padded shard of ``full`` (same device and dtype)."""
    L = shard_len(full.numel(), world_size)
    s = min(rank * L, full.numel())
    e = min(s + L, full.numel())
    out = torch.zeros(L, dtype=full.dtype, device=full.device)
    if e > s:
        out[: e - s].copy_(full[s:e])
    return out


def partition(full, world_size: int, tier: TierKind, store: TierStore, key: str | None = None,
              comm=None) -> PartitionedTensor:
    """write every (local) rank's shard to ``tier`` and flush."""
    t = _as_tensor(full)
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    key = key if key is not None else f"tensor{next(_auto_key)}"
    pt = PartitionedTensor(key, t.numel(), t.dtype, world_size, tier)
    tickets = [store.write(pt.shard_key(r), make_shard(t, world_size, r), tier)
               for r in _ranks(world_size, comm)]
    store.flush(tickets)
    return pt


# Pinned host staging buffers read by libzinf's asynchronous copies. torch's caching host
# allocator only tracks its own copies, so a buffer dropped right after the launch could
# be handed to the next NVMe read while the copy engine still reads it: keep each batch
# alive until an event recorded after its consumer has completed.
_inflight: list = []


def _keep_until_done(bufs) -> None:
    while _inflight and _inflight[0][0].query():
        _inflight.pop(0)
    ev = torch.cuda.Event()
    ev.record()
    _inflight.append((ev, bufs))


def _device_shard(pt: PartitionedTensor, store: TierStore, rank: int) -> torch.Tensor:
    """A tensor the gather can read directly: HBM or pinned host (UVA)."""
    k = pt.shard_key(rank)
    if not store.exists(k, pt.tier):
        from .store import KeyNotFound
        raise KeyNotFound(f"{k!r} not in {pt.tier.value} tier")
    if pt.tier is TierKind.NVME:
        return store.read(k, pt.tier).wait()       # pinned host staging
    t = store.tensor(k, pt.tier)
    store._note_read(pt.tier, t.numel() * t.element_size())
    return t


def allgather(pt: PartitionedTensor, store: TierStore, comm=None, out: torch.Tensor | None = None,
              use_copy_engine: bool = False, method: str = "p2p") -> torch.Tensor:
    """full tensor on the GPU, truncated to full_len.

    All shard reads are issued before the single gather (so NVMe reads run
    concurrently on the store's workers). Returns ``out``.
    """
    L = pt.shard_len
    if out is None:
        out = torch.empty(pt.full_len, dtype=pt.dtype, device=store.device)
    if out.numel() < pt.full_len or out.dtype != pt.dtype:
        raise ValueError("out too small or wrong dtype")
    if comm is None or comm.is_local:
        if pt.tier is TierKind.NVME:
            tickets = [store.read(pt.shard_key(r), pt.tier) for r in range(pt.world_size)]
            shards = [t.wait() for t in tickets]
        else:
            shards = [_device_shard(pt, store, r) for r in range(pt.world_size)]
        kernels.allgather(shards, L, out, pt.full_len,
                          use_copy_engine=use_copy_engine or pt.tier is not TierKind.DEVICE)
        if pt.tier is TierKind.NVME:
            _keep_until_done(shards)
        return out
    mine = _device_shard(pt, store, comm.rank)
    if method == "nccl":
        if not mine.is_cuda:
            mine = mine.to(store.device, non_blocking=True)
        padded = torch.empty(L * pt.world_size, dtype=pt.dtype, device=store.device)
        dist.all_gather_into_tensor(padded, mine, group=comm.group)
        out[: pt.full_len].copy_(padded[: pt.full_len])
        return out
    if method != "p2p":
        raise ValueError("method must be 'p2p' or 'nccl'")
    # one persistent shared window per PartitionedTensor: our shard is staged into it
    # (an H2D for host / NVMe tiers: the cg step), then every rank's window is read
    # over NVLink (the gg step) by the SM gather kernel or the copy engines
    stage, _ = comm.staging(f"ag:{pt.key}", L, pt.dtype)
    comm.device_barrier(channel=PARTITION_CHANNEL)   # peers finished reading the last gather
    stage.copy_(mine, non_blocking=True)
    comm.device_barrier(channel=PARTITION_CHANNEL)   # every rank's shard is staged
    comm.allgather_window(stage, L, out[: pt.full_len], use_copy_engine=use_copy_engine)
    return out


def reduce_scatter(contribs, world_size: int, comm=None, scale: float = 1.0,
                   ranks=None) -> list[torch.Tensor]:
    """shard r of the elementwise sum, folded in rank order.

    ``contribs``: full-length CUDA tensors in fold order. In the simulated
    model (no comm / LocalComm) they are every rank's contributions. With a
    DistComm they are this process's own contributions (one per rank in
    standard DP, or k per rank when a rank holds k fixed gradient groups):
    they are staged into a shared window and every rank's entries are read
    over NVLink, folded rank-major (rank 0's first, ... ) — the same order
    the simulated model uses. Half inputs produce fp32 shards (the cast of
    SPEC.md:782 fused in); f32 / f64 inputs keep their dtype. Returns the
    shards of ``ranks`` (default: every local rank).
    """
    contribs = [c if isinstance(c, int) else c.contiguous() for c in contribs]
    ref = next(c for c in contribs if not isinstance(c, int))
    n = ref.numel()
    for c in contribs:
        if not isinstance(c, int) and (c.numel() != n or c.dtype != ref.dtype):
            raise ValueError("all contribs must share length and dtype")
    L = shard_len(n, world_size)
    out_dt = torch.float64 if ref.dtype == torch.float64 else torch.float32
    rs = list(ranks) if ranks is not None else list(_ranks(world_size, comm))
    ptrs = [c if isinstance(c, int) else c.data_ptr() for c in contribs]
    dist_mode = comm is not None and not comm.is_local and comm.world > 1
    if dist_mode:
        if comm.world != world_size:
            raise ValueError("world_size disagrees with the communicator")
        k = len(contribs)
        stage, peer = comm.staging(f"rs:{n}:{k}", k * n, ref.dtype)
        comm.device_barrier(channel=PARTITION_CHANNEL)   # peers finished the last fold
        for j, c in enumerate(contribs):
            stage[j * n:(j + 1) * n].copy_(c, non_blocking=True)
        comm.device_barrier(channel=PARTITION_CHANNEL)   # every rank's contributions staged
        es = ref.element_size()
        ptrs = [p + j * n * es for p in peer for j in range(k)]
        rs = [comm.rank]
    outs = []
    arr = _lib.ptr_array(ptrs)
    stream = torch.cuda.current_stream().cuda_stream
    for r in rs:
        o = torch.empty(L, dtype=out_dt, device=ref.device)
        _lib.call("zi_reduce_scatter", arr, len(ptrs), r * L, L, n, _DT[ref.dtype], scale,
                  o.data_ptr(), stream)
        outs.append(o)
    return outs


def broadcast_fetch(key: str, tier: TierKind, store: TierStore, comm=None, owner: int = 0,
                    numel: int | None = None, dtype: torch.dtype | None = None
                    ) -> tuple[torch.Tensor, int]:
    """whole tensor from one owner key; all bytes on one path.

    Simulated ranks (no comm / LocalComm): the owner's store read, as the SPEC.
    With a DistComm the tensor lives only in ``owner``'s store: the owner
    stages it into a shared window and every rank pulls the whole tensor from
    that one GPU (copy engines) — the owner-broadcast baseline the
    bandwidth-centric all-gather replaces. Non-owners pass
    ``numel`` / ``dtype``. Returns (tensor, bytes charged to the owner's path).
    """
    if comm is None or comm.is_local or comm.world == 1:
        data = store.read(key, tier).wait()
        t = data if data.is_cuda else data.to(store.device, non_blocking=True)
        return t, t.numel() * t.element_size()
    if comm.rank == owner:
        data = store.read(key, tier).wait()
        numel, dtype = data.numel(), data.dtype
    elif numel is None or dtype is None:
        raise ValueError("non-owner ranks pass numel and dtype")
    stage, peer = comm.staging(f"bc:{key}", numel, dtype)
    comm.device_barrier(channel=PARTITION_CHANNEL)   # peers finished the last fetch
    if comm.rank == owner:
        stage[:numel].copy_(data, non_blocking=True)
    comm.device_barrier(channel=PARTITION_CHANNEL)   # the owner's copy is staged
    out = torch.empty(numel, dtype=dtype, device=store.device)
    kernels.allgather([peer[owner]], numel, out, numel, use_copy_engine=True)
    return out, numel * out.element_size() * (comm.world - 1)
