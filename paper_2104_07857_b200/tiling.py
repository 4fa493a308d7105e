"""Memory-centric tiling of large linear operators (PAPER §5.1.3).

A linear out_dim x in_dim is split into T row-block tiles (ceil split, a
possibly smaller last tile); each tile's [W_t, b_t] is one
PartitionedTensor in the tier store. ``forward_tiled`` runs the tiles
sequentially: fetch (all-gather of the tile's shards, prefetched one tile
ahead on a side stream) -> y_t = x W_t^T + b_t on the tcgen05 tensor cores
(zi_linear_fwd, bf16) -> release. ``backward_tiled`` re-fetches each tile
and produces dW_t = g_t^T x, db_t = sum g_t and the running
dx = sum_t g_t W_t.

Resident parameter memory is two tiles (the one computing + the one being
prefetched); ``prefetch=False`` gives the SPEC's strict one-tile bound
(SPEC.md:681). fp32 / fp64 tiles (the SPEC's f32/f64 equivalence checks)
run their products through cuBLAS; bf16 tiles use the libzinf kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import kernels
from .partition import PartitionedTensor, allgather, partition
from .store import TierKind, TierStore


def tile_rows(out_dim: int, tiles: int) -> list[tuple[int, int]]:
    """[(row_start, row_stop)]; T=4, out=10 -> rows (3,3,3,1)."""
    if tiles < 1:
        raise ValueError("T must be >= 1")
    R = -(-out_dim // tiles)
    out = []
    for t in range(tiles):
        s = min(t * R, out_dim)
        out.append((s, min(s + R, out_dim)))
    return out


@dataclass
class TiledLinear:
    """SPEC.md:631-636."""
    key: str
    in_dim: int
    out_dim: int
    tiles: int
    rows: list
    parts: list          # PartitionedTensor per non-empty tile (None for empty tiles)
    dtype: torch.dtype

    def tile_bytes(self, t: int) -> int:
        s, e = self.rows[t]
        return (e - s) * (self.in_dim + 1) * torch.empty(0, dtype=self.dtype).element_size()


def tile_linear(W: torch.Tensor, b: torch.Tensor, T: int, store: TierStore, tier: TierKind,
                key: str = "linear", world_size: int = 1, comm=None) -> TiledLinear:
    """persist T row-block tiles as partitioned [W_t, b_t] buckets."""
    out_dim, in_dim = W.shape
    if b.shape != (out_dim,):
        raise ValueError("bias length must equal out_dim")
    rows = tile_rows(out_dim, T)
    parts = []
    for t, (s, e) in enumerate(rows):
        if e <= s:
            parts.append(None)
            continue
        flat = torch.cat([W[s:e].reshape(-1), b[s:e]])
        parts.append(partition(flat, world_size, tier, store, key=f"{key}.tile{t}", comm=comm))
    return TiledLinear(key, in_dim, out_dim, T, rows, parts, W.dtype)


class _TileFetcher:
    """Two-slot ring of gathered tiles, filled on a side stream."""

    def __init__(self, tl: TiledLinear, store: TierStore, comm, prefetch: bool):
        self.tl, self.store, self.comm, self.prefetch = tl, store, comm, prefetch
        n = max((p.shard_len * p.world_size for p in tl.parts
                 if p is not None and not self._zero_copy(p)), default=1)
        self.slots = [torch.empty(n, dtype=tl.dtype, device=store.device) for _ in range(2)]
        self.stream = torch.cuda.Stream(store.device) if prefetch else None
        self.ready = {}
        self.peak_resident = 0

    def _zero_copy(self, p: PartitionedTensor) -> bool:
        # one rank holding the whole tile in HBM: the shard *is* the gathered tile
        return p.world_size == 1 and p.tier is TierKind.DEVICE and \
            (self.comm is None or self.comm.is_local)

    def issue(self, t: int) -> None:
        p: PartitionedTensor = self.tl.parts[t]
        if self._zero_copy(p):
            return
        slot = self.slots[t % 2]
        cur = torch.cuda.current_stream()
        if self.stream is None:
            allgather(p, self.store, self.comm, out=slot)
            return
        self.stream.wait_stream(cur)  # the slot's previous tile is no longer read
        with torch.cuda.stream(self.stream):
            allgather(p, self.store, self.comm, out=slot)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.ready[t] = ev

    def get(self, t: int):
        ev = self.ready.pop(t, None)
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)
        s, e = self.tl.rows[t]
        p = self.tl.parts[t]
        if self._zero_copy(p):
            flat = self.store.tensor(p.shard_key(0), p.tier)
        else:
            flat = self.slots[t % 2]
        live = 2 if self.prefetch else 1
        self.peak_resident = max(self.peak_resident, live * self.tl.tile_bytes(t))
        n = (e - s) * self.tl.in_dim
        return flat[:n].view(e - s, self.tl.in_dim), flat[n:n + (e - s)]


def _tiles(tl):
    return [t for t, p in enumerate(tl.parts) if p is not None]


def forward_tiled(tl: TiledLinear, x: torch.Tensor, store: TierStore, comm=None,
                  prefetch: bool = True, out: torch.Tensor | None = None,
                  fetcher: _TileFetcher | None = None) -> torch.Tensor:
    """y = concat_t(x W_t^T + b_t), tiles fetched/released in order."""
    if x.shape[-1] != tl.in_dim:
        raise ValueError("x width must equal in_dim")
    M = x.shape[0]
    y = out if out is not None else torch.empty(M, tl.out_dim, dtype=x.dtype, device=x.device)
    f = fetcher or _TileFetcher(tl, store, comm, prefetch)
    order = _tiles(tl)
    if order:
        f.issue(order[0])
    for i, t in enumerate(order):
        W_t, b_t = f.get(t)
        if i + 1 < len(order):
            f.issue(order[i + 1])
        s, e = tl.rows[t]
        if x.dtype == torch.bfloat16:
            kernels.linear_fwd(x, W_t, b_t, y[:, s:e])
        else:
            torch.addmm(b_t, x, W_t.t(), out=y[:, s:e]) if y[:, s:e].is_contiguous() else \
                y[:, s:e].copy_(torch.addmm(b_t, x, W_t.t()))
    forward_tiled.last_fetcher = f
    return y


def backward_tiled(tl: TiledLinear, x: torch.Tensor, gy: torch.Tensor, store: TierStore,
                   comm=None, prefetch: bool = True):
    """per tile dW_t = g_t^T x, db_t = sum g_t; dx = sum_t g_t W_t in tile order.

    Returns (dW tiles, db tiles, dx); empty tiles contribute nothing.
    """
    if gy.shape != (x.shape[0], tl.out_dim):
        raise ValueError("upstream grad shape mismatch")
    f = _TileFetcher(tl, store, comm, prefetch)
    order = _tiles(tl)
    dW, db = [None] * tl.tiles, [None] * tl.tiles
    acc_dt = torch.float32 if x.dtype in (torch.bfloat16, torch.float16) else x.dtype
    dx = torch.zeros(x.shape, dtype=acc_dt, device=x.device)
    if order:
        f.issue(order[0])
    for i, t in enumerate(order):
        W_t, _ = f.get(t)
        if i + 1 < len(order):
            f.issue(order[i + 1])
        s, e = tl.rows[t]
        g = gy[:, s:e]
        if x.dtype == torch.bfloat16:
            # zi_linear_tile_bwd on tcgen05: dW_t = g^T x, dx += g W_t (fp32 accumulate,
            # tiles in order), db_t = fixed-order column sums of g
            dW[t] = torch.empty(e - s, tl.in_dim, dtype=x.dtype, device=x.device)
            dbt = torch.empty(e - s, dtype=torch.float32, device=x.device)
            kernels.linear_tile_bwd(x, W_t, g, dw_t=dW[t], dx_acc=dx, db_t=dbt)
            db[t] = dbt.to(x.dtype)
        else:
            dW[t] = g.t() @ x
            dx += g @ W_t
            db[t] = g.sum(0)
    return dW, db, dx.to(x.dtype)
