"""CPU restatement of the partition-collectives module.

TEST INFRASTRUCTURE (see oracle/__init__.py). Ranks are indices in one
process exactly as the SPEC states; the GPU product runs one
process per GPU and must produce the same bytes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_len(full_len: int, world_size: int) -> int:
    """ceil(full_len / world_size)."""
    if full_len < 1 or world_size < 1:
        raise ValueError("need full_len >= 1 and world_size >= 1")
    return -(-full_len // world_size)


def shard_key(key: str, rank: int) -> str:
    """Per-rank shard key ``key + "/rank" + r``."""
    return f"{key}/rank{rank}"


def shard_range(full_len: int, world_size: int, rank: int) -> tuple[int, int, int]:
    """(start, stop, pad) of rank's slice of the full tensor."""
    L = shard_len(full_len, world_size)
    start = min(rank * L, full_len)
    stop = min(start + L, full_len)
    return start, stop, L - (stop - start)


@dataclass(frozen=True)
class PartitionedTensorRef:
    """SPEC.md:456-462 PartitionedTensor."""
    key: str
    full_len: int
    dtype: np.dtype
    world_size: int
    tier: str

    @property
    def shard_len(self) -> int:
        return shard_len(self.full_len, self.world_size)

    def shard_key(self, rank: int) -> str:
        return shard_key(self.key, rank)


def partition(full: np.ndarray, world_size: int) -> list[np.ndarray]:
    """ceil split, zero pad the final shard(s)."""
    full = np.asarray(full)
    if full.ndim != 1 or full.size == 0:
        raise ValueError("full must be a nonempty 1-D array")
    L = shard_len(full.size, world_size)
    padded = np.zeros(L * world_size, dtype=full.dtype)
    padded[: full.size] = full
    return [padded[r * L:(r + 1) * L].copy() for r in range(world_size)]


def allgather(shards: list[np.ndarray], full_len: int) -> np.ndarray:
    """concatenate shards in rank order, truncate to full_len."""
    return np.concatenate(shards)[:full_len].copy()


def reduce_scatter(contribs: list[np.ndarray], world_size: int,
                   acc_dtype=None) -> list[np.ndarray]:
    """shard r of the elementwise sum, summed in fixed rank order.

    ``acc_dtype`` widens each contribution before summing (the engine sums
    half gradients in fp32); default sums in the input dtype.
    Contributions shorter than world_size*shard_len are zero padded.
    """
    if len(contribs) != world_size:
        raise ValueError("need one contribution per rank")
    n = contribs[0].size
    for c in contribs:
        if c.size != n or c.dtype != contribs[0].dtype:
            raise ValueError("all contribs must share length and dtype")
    dt = np.dtype(acc_dtype) if acc_dtype is not None else contribs[0].dtype
    L = shard_len(n, world_size)
    s = np.zeros(L * world_size, dtype=dt)
    s[:n] = contribs[0].astype(dt)
    for k in range(1, world_size):
        t = np.zeros(L * world_size, dtype=dt)
        t[:n] = contribs[k].astype(dt)
        s = s + t
    return [s[r * L:(r + 1) * L].copy() for r in range(world_size)]


def reduce_scatter_cast(contribs_f32_of_half: list[np.ndarray], world_size: int,
                        scale: float) -> list[np.ndarray]:
    """The engine's fused RS: widen half contribs to fp32, rank-order sum, times scale.

    Mirrors kernel ``zi_reduce_scatter_cast``; inputs are the half values
    already widened to fp32 (exact), output fp32 shards.
    """
    shards = reduce_scatter([np.asarray(c, np.float32) for c in contribs_f32_of_half],
                            world_size, np.float32)
    sc = np.float32(scale)
    return [s * sc for s in shards]


def broadcast_fetch(full: np.ndarray) -> tuple[np.ndarray, int]:
    """same result as allgather; all bytes on one owner path."""
    full = np.asarray(full)
    return full.copy(), full.nbytes
