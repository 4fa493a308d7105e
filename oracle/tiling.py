"""CPU restatement of memory-centric tiling.

TEST INFRASTRUCTURE (see oracle/__init__.py). Tiles are row blocks of the
output dimension with a ceil split and a possibly smaller (or empty) last
tile; grad_x is a sequential running sum over tiles
(SPEC.md:662).
"""

from __future__ import annotations

import numpy as np


def tile_rows(out_dim: int, tiles: int) -> list[tuple[int, int]]:
    """[(row_start, row_stop)] per tile; T=4, out=10 -> rows (3,3,3,1)."""
    if tiles < 1:
        raise ValueError("T must be >= 1")
    R = -(-out_dim // tiles)
    out = []
    for t in range(tiles):
        s = min(t * R, out_dim)
        out.append((s, min(s + R, out_dim)))
    return out


def forward_tiled(W: np.ndarray, b: np.ndarray, x: np.ndarray, tiles: int) -> np.ndarray:
    """y_t = x W_t^T + b_t per tile, concatenated along features."""
    ys = []
    for s, e in tile_rows(W.shape[0], tiles):
        if e > s:
            ys.append(x @ W[s:e].T + b[s:e])
    return np.concatenate(ys, axis=-1)


def backward_tiled(W: np.ndarray, x: np.ndarray, gy: np.ndarray, tiles: int):
    """dW_t = g_t^T x, db_t = sum g_t, dx = sum_t g_t W_t (in tile order)."""
    dW = np.zeros_like(W)
    db = np.zeros(W.shape[0], dtype=W.dtype)
    dx = None
    for s, e in tile_rows(W.shape[0], tiles):
        if e <= s:
            continue
        g = gy[:, s:e]
        dW[s:e] = g.T @ x
        db[s:e] = g.sum(axis=0)
        part = g @ W[s:e]
        dx = part if dx is None else dx + part
    return dW, db, dx


def peak_tile_bytes(out_dim: int, in_dim: int, tiles: int, itemsize: int) -> int:
    """Largest resident tile (parameters) in bytes: ceil(out/T) rows."""
    return max(e - s for s, e in tile_rows(out_dim, tiles)) * in_dim * itemsize
