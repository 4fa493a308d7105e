"""CPU restatement of chunked mixed-precision Adam.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Every scalar is materialised as float32 exactly as the host passes it to the
CUDA kernel (``AdamConsts``), and every array operation is a single IEEE
float32 operation (numpy float32 + - * / sqrt are correctly rounded), in the
order the kernel issues its ``__f*_rn`` intrinsics. The kernel therefore
matches this function bit-for-bit:

    m  = b1*m + (1-b1)*g
    v  = b2*v + (1-b2)*(g*g)
    mh = m / (1-b1^t) ;  vh = v / (1-b2^t)
    p  = p - (lr*mh) / (sqrt(vh) + eps)          (no weight decay)
    p_half = RNE(p)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .numerics import f32_to_half_bits, half_bits_to_f32


@dataclass(frozen=True)
class AdamConsts:
    lr: np.float32
    b1: np.float32
    omb1: np.float32
    b2: np.float32
    omb2: np.float32
    bc1: np.float32
    bc2: np.float32
    eps: np.float32

    @staticmethod
    def make(lr: float, beta1: float, beta2: float, eps: float, step: int) -> "AdamConsts":
        """Host-side constant folding, identical to ``adam_consts`` in the product."""
        if step < 1:
            raise ValueError("Adam step counter starts at 1")
        f = np.float32
        return AdamConsts(f(lr), f(beta1), f(1.0 - beta1), f(beta2), f(1.0 - beta2),
                          f(1.0 - beta1 ** step), f(1.0 - beta2 ** step), f(eps))


def adam_update(p: np.ndarray, m: np.ndarray, v: np.ndarray, g: np.ndarray,
                c: AdamConsts) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """One elementwise Adam step on fp32 arrays; returns new (p, m, v)."""
    f32 = np.float32
    p = np.asarray(p, f32); m = np.asarray(m, f32); v = np.asarray(v, f32)
    g = np.asarray(g, f32)
    m2 = c.b1 * m + c.omb1 * g
    v2 = c.b2 * v + c.omb2 * (g * g)
    mh = m2 / c.bc1
    vh = v2 / c.bc2
    den = np.sqrt(vh) + c.eps
    p2 = p - (c.lr * mh) / den
    return p2.astype(f32), m2.astype(f32), v2.astype(f32)


def chunked_adam_step(p: np.ndarray, m: np.ndarray, v: np.ndarray, g: np.ndarray,
                      c: AdamConsts, chunk_elems: int, half_kind: int):
    """stream the shard chunk by chunk; returns (p, m, v, p_half_bits).

    Chunks never exceed ``chunk_elems``; the result is independent of it
    (elementwise).
    """
    if chunk_elems < 1:
        raise ValueError("chunk_elems must be >= 1")
    n = p.size
    P = np.empty(n, np.float32); M = np.empty(n, np.float32); V = np.empty(n, np.float32)
    H = np.empty(n, np.uint16)
    for s in range(0, n, chunk_elems):
        e = min(n, s + chunk_elems)
        P[s:e], M[s:e], V[s:e] = adam_update(p[s:e], m[s:e], v[s:e], g[s:e], c)
        H[s:e] = f32_to_half_bits(P[s:e], half_kind)
    return P, M, V, H


def rs_adam(p, m, v, contribs_half_bits: list[np.ndarray], rank: int, world: int,
            scale: float, c: AdamConsts, half_kind: int):
    """The engine's fused per-layer update (kernel ``zi_rs_adam``).

    g = (sum over ranks k=0..N-1, in order, of fp32(half contrib_k[shard r])) * scale,
    then ``adam_update`` and the RNE half param. Equal to reduce_scatter_cast
    followed by chunked_adam_step, by construction.
    """
    L = p.size
    g = np.zeros(L, np.float32)
    for k in range(world):
        seg = np.zeros(L, np.uint16)
        src = contribs_half_bits[k][rank * L:(rank + 1) * L]
        seg[: src.size] = src
        w = half_bits_to_f32(seg, half_kind)
        g = w.copy() if k == 0 else g + w
    g = g * np.float32(scale)
    P, M, V = adam_update(p, m, v, g, c)
    return P, M, V, f32_to_half_bits(P, half_kind), g
