"""The SPEC train-harness on B200: the reference-facing API of the engine.

Mixed-precision training of the SPEC's toy layered model under partitioned,
tier-placed model states, driven entirely through this package's drop-in
pieces — TierStore tiers, partition / allgather / reduce_scatter, the
prefetch plan, tiled linears and the libzinf Adam kernel:

* ``init_partitioned`` generates each layer on the GPU with the counter RNG
  (zi_init_uniform), partitions it immediately and discards the full copy
  (SPEC.md:727-735); tied pairs are wired with ``register_external_param``.
* ``train_step``: forward per layer = gather (fp16 -> fp32 widen) -> compute
  -> release; MSE loss; backward re-gathers, rounds each gradient group to
  half, reduce-scatters the G group contributions in fixed
  order (fp32 fold) and offloads the owned fp32 gradient shard
  to the placement tier; then ``chunked_adam_step`` streams every shard
  through the Adam kernel in chunks.

Bucket keys, init streams, gradient groups and digest follow
oracle/harness.py exactly, so results are world-size and placement
invariant bit-for-bit (AC-9) and match the oracle within fp32 tolerance.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

from . import _lib, kernels
from .partition import PartitionedTensor, allgather, partition, reduce_scatter
from .schedule import plan_prefetch, trace_schedule
from .store import KeyNotFound, TierKind, TierStore

ACTS = ("identity", "relu", "gelu-approx")


class MissingParam(KeyError):
    """A layer read a parameter outside its registered fetch set."""


@dataclass(frozen=True)
class LayerSpec:
    kind: str  # "linear" | "tiled_linear"
    in_dim: int
    out_dim: int
    act: str = "identity"
    tiles: int = 1


@dataclass
class ModelSpec:
    """SPEC.md:709-711."""
    layers: list
    tied_pairs: list = field(default_factory=list)
    seed: int = 7

    def __post_init__(self):
        for a, b in zip(self.layers, self.layers[1:]):
            if a.out_dim != b.in_dim:
                raise ValueError("consecutive layer dims must compose")
        for a, b in self.tied_pairs:
            la, lb = self.layers[a], self.layers[b]
            if (la.kind, la.in_dim, la.out_dim, la.tiles) != (lb.kind, lb.in_dim, lb.out_dim, lb.tiles):
                raise ValueError("tied layers must have identical shapes")

    def operators(self):
        keys = own_buckets(self)
        for i, L in enumerate(self.layers):
            yield (tuple(k for k, _, _ in keys[i]), 2 * (L.in_dim + 1) * L.out_dim,
                   2 * L.in_dim * L.out_dim)


@dataclass
class AdamHyper:
    """SPEC.md:721-724."""
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    step: int = 0


@dataclass
class HarnessPlacement:
    """Tier of each state class (grads default to the optimizer tier)."""
    params: TierKind = TierKind.DEVICE
    optim: TierKind = TierKind.DEVICE
    grads: TierKind | None = None

    @property
    def grad_tier(self) -> TierKind:
        return self.grads if self.grads is not None else self.optim

    @staticmethod
    def all(tier: TierKind) -> "HarnessPlacement":
        return HarnessPlacement(tier, tier, tier)


def tile_rows(out_dim: int, tiles: int):
    R = -(-out_dim // tiles)
    return [(min(t * R, out_dim), min(t * R + R, out_dim)) for t in range(tiles)]


def own_buckets(spec: ModelSpec) -> dict:
    """layer index -> [(bucket key, row_start, row_stop)] the layer's weights live in."""
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


@dataclass
class PartitionedModel:
    spec: ModelSpec
    world: int
    store: TierStore
    placement: HarnessPlacement
    half: torch.dtype
    parts: dict = field(default_factory=dict)       # bucket -> PartitionedTensor of p16
    fetch_sets: dict = field(default_factory=dict)  # layer -> set of bucket keys
    comm: object = None

    def retrace(self):
        self.fwd_seq, self.bwd_seq = trace_schedule(self.spec)
        self.plan = plan_prefetch(self.fwd_seq, (3, 2, 1))


def _key(seed: int, stream: int) -> int:
    from .gpt import _splitmix_key
    return _splitmix_key(seed, stream)


def init_partitioned(spec: ModelSpec, world_size: int, store: TierStore,
                     placement: HarnessPlacement | None = None,
                     half: torch.dtype = torch.float16, comm=None) -> PartitionedModel:
    """generate, partition and discard layer by layer."""
    placement = placement or HarnessPlacement()
    model = PartitionedModel(spec, world_size, store, placement, half, comm=comm)
    tied_b = {b for _, b in spec.tied_pairs}
    dev = store.device
    for i, L in enumerate(spec.layers):
        model.fetch_sets[i] = set()
        if i in tied_b:
            continue
        bound = 1.0 / (L.in_dim ** 0.5)
        scale = float(bound * 2.0 ** -24)
        W = torch.empty(L.out_dim * L.in_dim, dtype=torch.float32, device=dev)
        b = torch.empty(L.out_dim, dtype=torch.float32, device=dev)
        kernels.init_uniform(W, None, _key(spec.seed, 2 * i), 0, scale)
        kernels.init_uniform(b, None, _key(spec.seed, 2 * i + 1), 0, scale)
        W = W.view(L.out_dim, L.in_dim)
        for key, s, e in own_buckets(spec)[i]:
            master = torch.cat([W[s:e].reshape(-1), b[s:e]])
            h = torch.empty(master.numel(), dtype=half, device=dev)
            kernels.cast_f32_to_half(master, h)
            model.parts[key] = partition(h, world_size, placement.params, store, f"{key}.p16", comm)
            partition(master, world_size, placement.optim, store, f"{key}.p32", comm)
            z = torch.zeros_like(master)
            partition(z, world_size, placement.optim, store, f"{key}.m", comm)
            partition(z, world_size, placement.optim, store, f"{key}.v", comm)
        del W, b
    for i in range(len(spec.layers)):
        if i not in tied_b:
            model.fetch_sets[i].update(k for k, _, _ in own_buckets(spec)[i])
    for a, b in spec.tied_pairs:
        for key, _, _ in own_buckets(spec)[b]:
            register_external_param(model, key, b)
    model.retrace()
    return model


def register_external_param(model: PartitionedModel, key: str, consumer_layer: int) -> None:
    """add ``key`` to a consumer's fetch set (idempotent)."""
    if key not in model.parts:
        raise KeyError(f"unknown parameter key {key!r}")
    if not 0 <= consumer_layer < len(model.spec.layers):
        raise IndexError("consumer_layer out of range")
    model.fetch_sets[consumer_layer].add(key)
    model.retrace()


def _act_fwd(name, z):
    if name == "identity":
        return z
    if name == "relu":
        return torch.relu(z)
    return F.gelu(z, approximate="tanh")


def _act_bwd(name, z, g):
    if name == "identity":
        return g
    if name == "relu":
        return g * (z > 0).to(g.dtype)
    return torch.ops.aten.gelu_backward(g, z, approximate="tanh")


def _gather_widen(model: PartitionedModel, key: str) -> torch.Tensor:
    pt: PartitionedTensor = model.parts[key]
    h = allgather(pt, model.store, model.comm)
    w = torch.empty(pt.full_len, dtype=torch.float32, device=h.device)
    kernels.cast_half_to_f32(h[:pt.full_len], w)
    return w


def _layer_weights(model, i, fetched):
    L = model.spec.layers[i]
    Ws, bs = [], []
    for key, s, e in own_buckets(model.spec)[i]:
        if key not in model.fetch_sets[i]:
            raise MissingParam(f"layer {i} reads {key!r} outside its fetch set")
        flat = fetched[key]
        n = (e - s) * L.in_dim
        Ws.append(flat[:n].view(e - s, L.in_dim))
        bs.append(flat[n:n + e - s])
    return torch.cat(Ws, 0), torch.cat(bs)


def train_step(model: PartitionedModel, batch, hyper: AdamHyper, store: TierStore,
               chunk_elems: int = 1 << 20, grad_groups: int = 4) -> float:
    """SPEC.md:747-755; returns the loss."""
    spec, N, G = model.spec, model.world, grad_groups
    x, t = batch
    B = x.shape[0]
    if G % N or B % G:
        raise ValueError("need world | grad_groups and grad_groups | batch")
    rows = B // G
    norm = float(B * t.shape[1])
    nl = len(spec.layers)
    dist_mode = model.comm is not None and not model.comm.is_local and N > 1
    # data parallel: with one process per rank, rank r computes the G/N groups
    # [r*G/N, (r+1)*G/N); the reduce-scatter folds every rank's groups rank-major,
    # which is group order, so the result is the simulated model's bit for bit
    groups = range(model.comm.rank * (G // N), (model.comm.rank + 1) * (G // N)) \
        if dist_mode else range(G)
    # ---- forward: fetch -> compute -> release, per layer
    acts = {g: [x[g * rows:(g + 1) * rows].float()] for g in groups}
    zs = {g: [] for g in groups}
    for i in range(nl):
        fetched = {k: _gather_widen(model, k) for k in sorted(model.fetch_sets[i])}
        W, b = _layer_weights(model, i, fetched)
        for g in groups:
            z = kernels.matmul_fixed(acts[g][-1], W.t(), bias=b)
            zs[g].append(z)
            acts[g].append(_act_fwd(spec.layers[i].act, z))
        del fetched, W, b  # release
    losses = []
    grads_out = {}
    for g in groups:
        d = acts[g][-1] - t[g * rows:(g + 1) * rows].float()
        losses.append((d * d).sum() / norm)
        grads_out[g] = 2.0 * d / norm
    if dist_mode:   # every group's loss, folded in group order in fp32 as below
        import numpy as np
        vals = [v for part in model.comm.all_gather_object([float(l.item()) for l in losses])
                for v in part]
        acc32 = np.float32(vals[0])
        for v in vals[1:]:
            acc32 = np.float32(acc32 + np.float32(v))
        loss = torch.tensor(float(acc32))
    else:
        loss = losses[0]
        for l in losses[1:]:
            loss = loss + l
    # ---- backward: re-gather, per-group grads, reduce + offload when a bucket completes
    last_use = {}
    for i in range(nl):
        for k, _, _ in own_buckets(spec)[i]:
            last_use.setdefault(k, i)   # first forward consumer = last backward consumer
    acc = {}
    for i in reversed(range(nl)):
        L = spec.layers[i]
        fetched = {k: _gather_widen(model, k) for k in sorted(model.fetch_sets[i])}
        W, _ = _layer_weights(model, i, fetched)
        for g in groups:
            dz = _act_bwd(L.act, zs[g][i], grads_out[g])
            dW = kernels.matmul_fixed(dz.t(), acts[g][i])
            db = dz.sum(0)
            grads_out[g] = kernels.matmul_fixed(dz, W)
            for key, s, e in own_buckets(spec)[i]:
                flat = torch.cat([dW[s:e].reshape(-1), db[s:e]])
                acc[(key, g)] = flat if (key, g) not in acc else acc[(key, g)] + flat
        del fetched, W
        for key, _, _ in own_buckets(spec)[i]:
            if last_use[key] == i:
                _reduce_offload(model, key, [acc.pop((key, g)) for g in groups], store)
    chunked_adam_step(model, hyper, chunk_elems, store)
    return float(loss.item())


def _reduce_offload(model: PartitionedModel, key: str, group_grads, store: TierStore) -> None:
    """Round each group gradient to half, fold in group order (fp32), offload owned shards."""
    pt = model.parts[key]
    contribs = []
    for gg in group_grads:
        h = torch.empty(gg.numel(), dtype=model.half, device=gg.device)
        kernels.cast_f32_to_half(gg.contiguous(), h)
        contribs.append(h)
    local = model.comm is None or model.comm.is_local
    ranks = range(model.world) if local else [model.comm.rank]
    # simulated ranks: every group is local; DistComm: this rank's groups, folded with
    # the peers' over NVLink (partition.reduce_scatter's shared window)
    shards = reduce_scatter(contribs, pt.world_size, comm=None if local else model.comm,
                            ranks=ranks)
    tickets = [store.write(f"{key}.g32/rank{r}", s, model.placement.grad_tier)
               for r, s in zip(ranks, shards)]
    store.flush(tickets)


def _to_dev(t: torch.Tensor, dev) -> torch.Tensor:
    return t if t.is_cuda else t.to(dev, non_blocking=True)


def chunked_adam_step(model: PartitionedModel, hyper: AdamHyper, chunk_elems: int,
                      store: TierStore) -> None:
    """stream master/m/v/grad chunks through zi_adam_step."""
    if chunk_elems < 1:
        raise ValueError("chunk_elems must be >= 1")
    hyper.step += 1
    c = _lib.adam_consts(hyper.lr, hyper.beta1, hyper.beta2, hyper.eps, hyper.step)
    opt, par, gt = model.placement.optim, model.placement.params, model.placement.grad_tier
    dev = store.device
    ranks = range(model.world) if (model.comm is None or model.comm.is_local) else [model.comm.rank]
    for key, pt in model.parts.items():
        for r in ranks:
            L = pt.shard_len
            for s in range(0, L, chunk_elems):
                n = min(chunk_elems, L - s)
                tk = [store.read_range(f"{key}.{nm}/rank{r}", tier, s, n)
                      for nm, tier in (("p32", opt), ("m", opt), ("v", opt), ("g32", gt))]
                p, m, v, g = (_to_dev(t.wait(), dev).clone() for t in tk)
                h = torch.empty(n, dtype=model.half, device=dev)
                kernels.adam_step(p, m, v, g, h, c)
                store.flush([store.write_range(f"{key}.p32/rank{r}", opt, s, p),
                             store.write_range(f"{key}.m/rank{r}", opt, s, m),
                             store.write_range(f"{key}.v/rank{r}", opt, s, v),
                             store.write_range(f"{key}.p16/rank{r}", par, s, h)])


def synthetic_batch(spec: ModelSpec, batch: int, device):
    """Same regression task as oracle/harness.py:synthetic_batch (counter RNG)."""
    d_in, d_out = spec.layers[0].in_dim, spec.layers[-1].out_dim
    x = torch.empty(batch * d_in, dtype=torch.float32, device=device)
    A = torch.empty(d_out * d_in, dtype=torch.float32, device=device)
    kernels.init_uniform(x, None, _key(spec.seed, 1000), 0, float(2.0 ** -24))
    kernels.init_uniform(A, None, _key(spec.seed, 1001), 0, float(2.0 ** -24))
    x = x.view(batch, d_in)
    return x, kernels.matmul_fixed(x, A.view(d_out, d_in).t())


def digest(model: PartitionedModel) -> str:
    """sha256 over sorted bucket keys + gathered fp32 master bytes (as the oracle)."""
    h = hashlib.sha256()
    for key in sorted(model.parts):
        pt = model.parts[key]
        p32 = PartitionedTensor(f"{key}.p32", pt.full_len, torch.float32, pt.world_size,
                                model.placement.optim)
        full = allgather(p32, model.store, model.comm)[:pt.full_len]
        h.update(key.encode() + b"\0")
        h.update(full.cpu().numpy().astype("<f4").tobytes())
    return h.hexdigest()


def run_training(spec: ModelSpec, world: int, placement: HarnessPlacement | None, steps: int,
                 seed: int | None, store: TierStore, batch: int = 16, lr: float = 1e-2,
                 half: torch.dtype = torch.float16, chunk_elems: int = 1 << 20, comm=None):
    """returns (digest, loss history).

    With a DistComm (one process per rank) each process passes its own store;
    the digest is identical on every rank and to the simulated run's."""
    if seed is not None:
        spec = ModelSpec(spec.layers, spec.tied_pairs, seed)
    model = init_partitioned(spec, world, store, placement, half, comm=comm)
    x, t = synthetic_batch(spec, batch, store.device)
    hyper = AdamHyper(lr=lr)
    losses = [train_step(model, (x, t), hyper, store, chunk_elems) for _ in range(steps)]
    return digest(model), losses
