"""CPU restatement of the SPEC train-harness on the toy layered model.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Conventions shared with the product engine
(``paper_2104_07857_b200.harness``), all stated in DESIGN.md:

* One PartitionedTensor per layer bucket: ``layer{i}`` = [W.ravel(), b]
  (block-flattening, the alternative SPEC.md:524 names). Tiled layers hold
  one bucket per tile, ``layer{i}.tile{t}`` = [W_t.ravel(), b_t].
* Init: W ~ counter-RNG stream 2i, b ~ stream 2i+1, both U(+-1/sqrt(in))
  generated in fp32; master = fp32 value, working copy = RNE half.
* Data parallel: the global batch is split into G equal contiguous row
  groups (G fixed, default 4), G/N per rank; per-group gradients are
  normalised by the global element count, rounded to half and
  reduce-scattered as a fold in global group order in fp32;
  scale 1. This makes results world-size invariant (AC-9).
* Tied pair (a, b): layer b consumes layer a's bucket;
  its gradient is accumulated in fp32 in backward order before the cast.
* Digest: sha256 over sorted bucket keys + gathered fp32 master bytes.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

from . import numerics as nx
from .adam import AdamConsts, chunked_adam_step
from .partition import allgather, partition, reduce_scatter
from .tiling import tile_rows

ACTS = ("identity", "relu", "gelu-approx")


@dataclass(frozen=True)
class LayerSpec:
    kind: str  # "linear" | "tiled_linear"
    in_dim: int
    out_dim: int
    act: str = "identity"
    tiles: int = 1


@dataclass
class ModelSpec:
    layers: list
    tied_pairs: list = field(default_factory=list)
    seed: int = 7


def bucket_keys(spec: ModelSpec) -> dict:
    """layer index -> list of (bucket key, row_start, row_stop) it consumes."""
    owner = {b: a for a, b in spec.tied_pairs}
    out = {}
    for i, L in enumerate(spec.layers):
        src = owner.get(i, i)
        if L.kind == "tiled_linear":
            out[i] = [(f"layer{src}.tile{t}", s, e)
                      for t, (s, e) in enumerate(tile_rows(L.out_dim, L.tiles)) if e > s]
        else:
            out[i] = [(f"layer{src}", 0, L.out_dim)]
    return out


def init_layer_fp32(spec: ModelSpec, i: int):
    L = spec.layers[i]
    bound = nx.init_bound(L.in_dim)
    W = nx.uniform_init(spec.seed, 2 * i, 0, L.out_dim * L.in_dim, bound).reshape(L.out_dim, L.in_dim)
    b = nx.uniform_init(spec.seed, 2 * i + 1, 0, L.out_dim, bound)
    return W, b


def init_buckets(spec: ModelSpec) -> dict:
    """bucket key -> fp32 master flat vector (owner layers only)."""
    owners = {b for _, b in spec.tied_pairs}
    out = {}
    for i, L in enumerate(spec.layers):
        if i in owners:
            continue
        W, b = init_layer_fp32(spec, i)
        if L.kind == "tiled_linear":
            for t, (s, e) in enumerate(tile_rows(L.out_dim, L.tiles)):
                if e > s:
                    out[f"layer{i}.tile{t}"] = np.concatenate([W[s:e].ravel(), b[s:e]])
        else:
            out[f"layer{i}"] = np.concatenate([W.ravel(), b])
    return out


def act_fwd(name: str, z):
    if name == "identity":
        return z
    if name == "relu":
        return np.maximum(z, 0)
    if name == "gelu-approx":
        t = z.dtype.type
        c = t(np.sqrt(2.0 / np.pi))
        return t(0.5) * z * (1 + np.tanh(c * (z + t(0.044715) * z * z * z)))
    raise ValueError(name)


def act_bwd(name: str, z, g):
    if name == "identity":
        return g
    if name == "relu":
        return g * (z > 0).astype(z.dtype)
    if name == "gelu-approx":
        t = z.dtype.type
        c = t(np.sqrt(2.0 / np.pi))
        u = c * (z + t(0.044715) * z * z * z)
        th = np.tanh(u)
        du = c * (1 + t(3 * 0.044715) * z * z)
        return g * (t(0.5) * (1 + th) + t(0.5) * z * (1 - th * th) * du)
    raise ValueError(name)


def unpack(spec: ModelSpec, i: int, buckets: dict, dtype):
    """Widened (W, b) of layer i from the gathered half buckets it consumes."""
    L = spec.layers[i]
    Ws, bs = [], []
    for key, s, e in bucket_keys(spec)[i]:
        flat = buckets[key].astype(dtype)
        rows = e - s
        Ws.append(flat[: rows * L.in_dim].reshape(rows, L.in_dim))
        bs.append(flat[rows * L.in_dim:])
    return np.concatenate(Ws, 0), np.concatenate(bs)


def forward_backward(spec: ModelSpec, buckets: dict, x, t, norm: float, dtype=np.float32):
    """Loss contribution and fp32 (or f64) bucket grads for one rank's rows.

    ``buckets`` are widened gathered params (key -> flat). Loss = sum of squared
    error / norm; grads accumulate per bucket in backward order.
    """
    a = x.astype(dtype)
    saved = []
    for i, L in enumerate(spec.layers):
        W, b = unpack(spec, i, buckets, dtype)
        z = a @ W.T + b
        saved.append((a, z, W))
        a = act_fwd(L.act, z)
    diff = a - t.astype(dtype)
    loss = (diff * diff).sum(dtype=dtype) / dtype(norm)
    g = dtype(2.0) * diff / dtype(norm)
    grads: dict = {}
    for i in reversed(range(len(spec.layers))):
        L = spec.layers[i]
        a_in, z, W = saved[i]
        dz = act_bwd(L.act, z, g)
        dW = dz.T @ a_in
        db = dz.sum(axis=0)
        g = dz @ W
        for key, s, e in bucket_keys(spec)[i]:
            flat = np.concatenate([dW[s:e].ravel(), db[s:e]])
            grads[key] = flat if key not in grads else grads[key] + flat
    return loss, grads


def synthetic_batch(spec: ModelSpec, batch: int):
    """Seeded regression task: x ~ U(-1,1), targets from a fixed linear teacher."""
    d_in, d_out = spec.layers[0].in_dim, spec.layers[-1].out_dim
    x = nx.uniform_init(spec.seed, 1000, 0, batch * d_in, 1.0).reshape(batch, d_in)
    A = nx.uniform_init(spec.seed, 1001, 0, d_out * d_in, 1.0).reshape(d_out, d_in)
    return x, (x @ A.T).astype(np.float32)


@dataclass
class OracleState:
    """Per-bucket, per-rank shards: p16 (half bits), p32, m, v."""
    world: int
    half_kind: int
    full_len: dict
    p16: dict
    p32: dict
    m: dict
    v: dict
    step: int = 0


def init_partitioned(spec: ModelSpec, world: int, half_kind: int = nx.HALF_FP16) -> OracleState:
    """SPEC.md:727-735."""
    st = OracleState(world, half_kind, {}, {}, {}, {}, {})
    for key, full in init_buckets(spec).items():
        st.full_len[key] = full.size
        st.p32[key] = partition(full, world)
        st.p16[key] = [nx.f32_to_half_bits(s, half_kind) for s in st.p32[key]]
        st.m[key] = [np.zeros_like(s) for s in st.p32[key]]
        st.v[key] = [np.zeros_like(s) for s in st.p32[key]]
    return st


def gathered_half(st: OracleState) -> dict:
    return {k: nx.half_bits_to_f32(allgather(st.p16[k], st.full_len[k]), st.half_kind)
            for k in st.p16}


def train_step(spec: ModelSpec, st: OracleState, x, t, lr=1e-2, betas=(0.9, 0.999),
               eps=1e-8, chunk_elems=1 << 20, grad_groups: int = 4) -> float:
    """SPEC.md:747-755. Returns the global loss.

    The batch is cut into ``grad_groups`` (G) equal row groups; rank r owns
    groups [r*G/N, (r+1)*G/N). Each group's gradient is rounded to half on its
    own and the reduce-scatter folds all G half contributions in global group
    order in fp32 — the "fixed rank order" sum of SPEC.md:487 with the group as
    the unit — and the loss is the fp32 fold of the G group losses. Because
    no partial sum depends on N, loss history and master params are
    bit-identical for every world size dividing G (AC-9).
    """
    N = st.world
    B = x.shape[0]
    G = grad_groups
    if G % N or B % G:
        raise ValueError("need world | grad_groups and grad_groups | batch")
    rows = B // G
    norm = float(B * t.shape[1])
    params = gathered_half(st)
    losses = []
    contribs: dict = {k: [] for k in st.p16}
    for g in range(G):  # rank r = g // (G // N) computes group g
        lg, gr = forward_backward(spec, params, x[g * rows:(g + 1) * rows],
                                  t[g * rows:(g + 1) * rows], norm)
        losses.append(np.float32(lg))
        for k in st.p16:
            contribs[k].append(nx.round_half(gr[k].astype(np.float32), st.half_kind))
    loss = losses[0]
    for lg in losses[1:]:
        loss = np.float32(loss + lg)
    st.step += 1
    c = AdamConsts.make(lr, betas[0], betas[1], eps, st.step)
    for k in st.p16:
        folded = reduce_scatter(contribs[k], G, np.float32)  # fold over G groups
        flat = np.concatenate(folded)[: st.full_len[k]]
        shards = partition(flat, N)
        for r in range(N):
            P, M, V, H = chunked_adam_step(st.p32[k][r], st.m[k][r], st.v[k][r], shards[r],
                                           c, chunk_elems, st.half_kind)
            st.p32[k][r], st.m[k][r], st.v[k][r], st.p16[k][r] = P, M, V, H
    return float(loss)


def digest(st: OracleState) -> str:
    h = hashlib.sha256()
    for k in sorted(st.p32):
        h.update(k.encode() + b"\0")
        h.update(allgather(st.p32[k], st.full_len[k]).astype("<f4").tobytes())
    return h.hexdigest()


def run_training(spec: ModelSpec, world: int, steps: int, batch: int = 16, lr=1e-2,
                 half_kind: int = nx.HALF_FP16, chunk_elems: int = 1 << 20):
    """returns (digest, loss history)."""
    st = init_partitioned(spec, world, half_kind)
    x, t = synthetic_batch(spec, batch)
    losses = [train_step(spec, st, x, t, lr=lr, chunk_elems=chunk_elems) for _ in range(steps)]
    return digest(st), losses
