"""GPT-block generalisation of the SPEC train_step (BASELINE configs 1-5).

TEST INFRASTRUCTURE (see oracle/__init__.py). numpy forward/backward of a
pre-LayerNorm GPT with a tied embedding, partitioned ZeRO-3 style exactly
like the SPEC harness:

* operators: op 0 ``embed`` (bucket "embed" = [wte, wpe]); ops 1..nl
  ``layer{i}`` (bucket "h{i}"); op nl+1 ``head`` (bucket "final" = [lnf_w,
  lnf_b] plus the external parameter "embed" — the tied embedding registered
  with register_external_param, PAPER §7.1.1).
* each bucket is one PartitionedTensor (ceil split, zero pad).
* init: counter RNG stream = op*64 + param index, U(+-1/sqrt(fan_in)) for
  matrices, 1/0 for LayerNorm, 0 for biases; fp32 master, RNE half copy.
* per-rank loss = mean token cross-entropy of the rank's micro-batch; grads
  rounded to half per contribution and reduce-scattered as an fp32 fold in
  rank order, scaled by 1/G (G = contribution count = world size).
* Adam as in oracle.adam (bit-exact restatement of the kernel).

Compute is fp32 (``dtype`` may be float64 for finite-difference checks).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import numerics as nx
from .adam import AdamConsts, adam_update
from .partition import allgather, partition, reduce_scatter

LN_EPS = 1e-5


@dataclass(frozen=True)
class GPTConfig:
    nl: int = 4
    hd: int = 256
    heads: int = 4
    seq: int = 128
    vocab: int = 512
    batch: int = 4          # per-rank micro-batch (sequences)

    @property
    def head_dim(self) -> int:
        return self.hd // self.heads


TINY = GPTConfig()                                                          # BASELINE config 1
GPT_1P3B = GPTConfig(nl=24, hd=2048, heads=16, seq=1024, vocab=50304, batch=8)  # config 2
GPT_10B = GPTConfig(nl=50, hd=4096, heads=32, seq=1024, vocab=50304, batch=8)   # config 3
GPT_70B = GPTConfig(nl=87, hd=8192, heads=64, seq=1024, vocab=50304, batch=4)   # config 5


def layer_params(c: GPTConfig):
    """[(name, shape, init)] of one transformer block; init = ("u", bound) | ("c", value)."""
    h = c.hd
    ub = ("u", nx.init_bound(h))
    return [
        ("ln1_w", (h,), ("c", 1.0)), ("ln1_b", (h,), ("c", 0.0)),
        ("qkv_w", (3 * h, h), ub), ("qkv_b", (3 * h,), ("c", 0.0)),
        ("proj_w", (h, h), ub), ("proj_b", (h,), ("c", 0.0)),
        ("ln2_w", (h,), ("c", 1.0)), ("ln2_b", (h,), ("c", 0.0)),
        ("fc1_w", (4 * h, h), ub), ("fc1_b", (4 * h,), ("c", 0.0)),
        ("fc2_w", (h, 4 * h), ("u", nx.init_bound(4 * h))), ("fc2_b", (h,), ("c", 0.0)),
    ]


def embed_params(c: GPTConfig):
    ub = ("u", nx.init_bound(c.hd))
    return [("wte", (c.vocab, c.hd), ub), ("wpe", (c.seq, c.hd), ub)]


def final_params(c: GPTConfig):
    return [("lnf_w", (c.hd,), ("c", 1.0)), ("lnf_b", (c.hd,), ("c", 0.0))]


def buckets(c: GPTConfig):
    """[(op index, bucket key, param list)] in forward op order."""
    out = [(0, "embed", embed_params(c))]
    for i in range(c.nl):
        out.append((i + 1, f"h{i}", layer_params(c)))
    out.append((c.nl + 1, "final", final_params(c)))
    return out


def bucket_numel(params) -> int:
    return sum(int(np.prod(s)) for _, s, _ in params)


def param_count(c: GPTConfig) -> int:
    return sum(bucket_numel(p) for _, _, p in buckets(c))


def bucket_segments(op: int, params):
    """[(offset, count, stream, init)] of a bucket; the generator's element index
    is the position inside the parameter tensor."""
    segs, off = [], 0
    for j, (_, shape, init) in enumerate(params):
        n = int(np.prod(shape))
        segs.append((off, n, op * 64 + j, init))
        off += n
    return segs


def init_bucket_range(seed: int, op: int, params, start: int, count: int) -> np.ndarray:
    """fp32 master values of bucket elements [start, start+count) — shard-local init."""
    out = np.zeros(count, np.float32)
    for off, n, stream, init in bucket_segments(op, params):
        s, e = max(start, off), min(start + count, off + n)
        if s >= e:
            continue
        if init[0] == "u":
            out[s - start:e - start] = nx.uniform_init(seed, stream, s - off, e - s, init[1])
        else:
            out[s - start:e - start] = np.float32(init[1])
    return out


def unflatten(flat: np.ndarray, params) -> dict:
    out, off = {}, 0
    for name, shape, _ in params:
        n = int(np.prod(shape))
        out[name] = flat[off:off + n].reshape(shape)
        off += n
    return out


def flatten(grads: dict, params, dtype=np.float32) -> np.ndarray:
    return np.concatenate([np.asarray(grads[name], dtype).ravel() for name, _, _ in params])


# ------------------------------------------------------------------ numerics

def ln_fwd(x, w, b):
    t = x.dtype.type
    mu = x.mean(-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdims=True)
    rstd = t(1.0) / np.sqrt(var + t(LN_EPS))
    xh = xc * rstd
    return xh * w + b, (xh, rstd)


def ln_bwd(dy, w, cache):
    xh, rstd = cache
    dw = (dy * xh).reshape(-1, xh.shape[-1]).sum(0)
    db = dy.reshape(-1, dy.shape[-1]).sum(0)
    dxh = dy * w
    dx = rstd * (dxh - dxh.mean(-1, keepdims=True) - xh * (dxh * xh).mean(-1, keepdims=True))
    return dx, dw, db


def gelu_fwd(z):
    t = z.dtype.type
    c = t(np.sqrt(2.0 / np.pi))
    return t(0.5) * z * (t(1) + np.tanh(c * (z + t(0.044715) * z * z * z)))


def gelu_bwd(z, g):
    t = z.dtype.type
    c = t(np.sqrt(2.0 / np.pi))
    th = np.tanh(c * (z + t(0.044715) * z * z * z))
    du = c * (t(1) + t(3 * 0.044715) * z * z)
    return g * (t(0.5) * (t(1) + th) + t(0.5) * z * (t(1) - th * th) * du)


def attn_fwd(qkv, c: GPTConfig):
    B, S, _ = qkv.shape
    H, D = c.heads, c.head_dim
    q, k, v = [qkv[:, :, i * c.hd:(i + 1) * c.hd].reshape(B, S, H, D).transpose(0, 2, 1, 3)
               for i in range(3)]
    t = qkv.dtype.type
    sc = t(1.0 / np.sqrt(D))
    s = (q @ k.transpose(0, 1, 3, 2)) * sc
    mask = np.triu(np.ones((S, S), bool), 1)
    s = np.where(mask, t(-np.inf), s)
    s = s - s.max(-1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(-1, keepdims=True)
    o = p @ v
    return o.transpose(0, 2, 1, 3).reshape(B, S, c.hd), (q, k, v, p)


def attn_bwd(do, cache, c: GPTConfig):
    q, k, v, p = cache
    B, H, S, D = q.shape
    t = q.dtype.type
    sc = t(1.0 / np.sqrt(D))
    do = do.reshape(B, S, H, D).transpose(0, 2, 1, 3)
    dv = p.transpose(0, 1, 3, 2) @ do
    dp = do @ v.transpose(0, 1, 3, 2)
    ds = p * (dp - (dp * p).sum(-1, keepdims=True))
    dq = (ds @ k) * sc
    dk = (ds.transpose(0, 1, 3, 2) @ q) * sc
    back = lambda x: x.transpose(0, 2, 1, 3).reshape(B, S, H * D)
    return np.concatenate([back(dq), back(dk), back(dv)], -1)


def block_fwd(x, P, c: GPTConfig):
    h1, ln1c = ln_fwd(x, P["ln1_w"], P["ln1_b"])
    qkv = h1 @ P["qkv_w"].T + P["qkv_b"]
    o, ac = attn_fwd(qkv, c)
    x2 = x + o @ P["proj_w"].T + P["proj_b"]
    h2, ln2c = ln_fwd(x2, P["ln2_w"], P["ln2_b"])
    u = h2 @ P["fc1_w"].T + P["fc1_b"]
    a = gelu_fwd(u)
    y = x2 + a @ P["fc2_w"].T + P["fc2_b"]
    return y, (x, h1, ln1c, ac, o, x2, h2, ln2c, u, a)


def block_bwd(dy, P, cache, c: GPTConfig):
    x, h1, ln1c, ac, o, x2, h2, ln2c, u, a = cache
    hd = c.hd
    g = {}
    dyf = dy.reshape(-1, hd)
    g["fc2_w"] = dyf.T @ a.reshape(-1, 4 * hd)
    g["fc2_b"] = dyf.sum(0)
    da = dy @ P["fc2_w"]
    du = gelu_bwd(u, da)
    duf = du.reshape(-1, 4 * hd)
    g["fc1_w"] = duf.T @ h2.reshape(-1, hd)
    g["fc1_b"] = duf.sum(0)
    dh2 = du @ P["fc1_w"]
    dx2, g["ln2_w"], g["ln2_b"] = ln_bwd(dh2, P["ln2_w"], ln2c)
    dx2 = dx2 + dy
    dx2f = dx2.reshape(-1, hd)
    g["proj_w"] = dx2f.T @ o.reshape(-1, hd)
    g["proj_b"] = dx2f.sum(0)
    do = dx2 @ P["proj_w"]
    dqkv = attn_bwd(do, ac, c)
    dqf = dqkv.reshape(-1, 3 * hd)
    g["qkv_w"] = dqf.T @ h1.reshape(-1, hd)
    g["qkv_b"] = dqf.sum(0)
    dh1 = dqkv @ P["qkv_w"]
    dx, g["ln1_w"], g["ln1_b"] = ln_bwd(dh1, P["ln1_w"], ln1c)
    return dx + dx2, g


def forward_backward(c: GPTConfig, full: dict, tokens: np.ndarray, targets: np.ndarray,
                     dtype=np.float32):
    """Loss (mean CE over the micro-batch) and per-bucket grads (fp32/f64 flats).

    ``full`` maps bucket key -> widened gathered flat vector.
    """
    t = dtype
    E = unflatten(full["embed"].astype(t), embed_params(c))
    B, S = tokens.shape
    x = E["wte"][tokens] + E["wpe"][:S]
    caches = []
    for i in range(c.nl):
        P = unflatten(full[f"h{i}"].astype(t), layer_params(c))
        x, cache = block_fwd(x, P, c)
        caches.append((P, cache))
    F = unflatten(full["final"].astype(t), final_params(c))
    hf, lnfc = ln_fwd(x, F["lnf_w"], F["lnf_b"])
    logits = hf.reshape(-1, c.hd) @ E["wte"].T
    mx = logits.max(-1, keepdims=True)
    ex = np.exp(logits - mx)
    se = ex.sum(-1, keepdims=True)
    tgt = targets.reshape(-1)
    T = tgt.size
    logp_t = (logits - mx - np.log(se))[np.arange(T), tgt]
    loss = -logp_t.sum(dtype=t) / t(T)
    # backward
    dlog = ex / se
    dlog[np.arange(T), tgt] -= t(1)
    dlog = dlog / t(T)
    grads = {}
    dwte = dlog.T @ hf.reshape(-1, c.hd)                     # head contribution first
    dhf = (dlog @ E["wte"]).reshape(B, S, c.hd)
    dx, dlnw, dlnb = ln_bwd(dhf, F["lnf_w"], lnfc)
    grads["final"] = flatten({"lnf_w": dlnw, "lnf_b": dlnb}, final_params(c), t)
    for i in reversed(range(c.nl)):
        P, cache = caches[i]
        dx, g = block_bwd(dx, P, cache, c)
        grads[f"h{i}"] = flatten(g, layer_params(c), t)
    demb = np.zeros_like(E["wte"])
    np.add.at(demb, tokens.reshape(-1), dx.reshape(-1, c.hd))
    dwte = dwte + demb
    dwpe = np.zeros_like(E["wpe"])
    dwpe[:S] = dx.sum(0)
    grads["embed"] = flatten({"wte": dwte, "wpe": dwpe}, embed_params(c), t)
    return loss, grads


def synthetic_tokens(c: GPTConfig, seed: int, rank: int, step: int = 0):
    """Token ids uniform on [0, V), per (rank, step); returns (inputs, targets)."""
    rng = np.random.default_rng([seed, rank, step])
    tok = rng.integers(0, c.vocab, size=(c.batch, c.seq + 1), dtype=np.int64)
    return tok[:, :-1].copy(), tok[:, 1:].copy()


@dataclass
class GPTOracleState:
    cfg: GPTConfig
    world: int
    half_kind: int
    seed: int
    full_len: dict
    p16: dict
    p32: dict
    m: dict
    v: dict
    step: int = 0


def init_partitioned(c: GPTConfig, world: int, seed: int = 7,
                     half_kind: int = nx.HALF_BF16) -> GPTOracleState:
    st = GPTOracleState(c, world, half_kind, seed, {}, {}, {}, {}, {})
    for op, key, params in buckets(c):
        n = bucket_numel(params)
        full = init_bucket_range(seed, op, params, 0, n)
        st.full_len[key] = n
        st.p32[key] = partition(full, world)
        st.p16[key] = [nx.f32_to_half_bits(s, half_kind) for s in st.p32[key]]
        st.m[key] = [np.zeros_like(s) for s in st.p32[key]]
        st.v[key] = [np.zeros_like(s) for s in st.p32[key]]
    return st


def gathered(st: GPTOracleState) -> dict:
    return {k: nx.half_bits_to_f32(allgather(st.p16[k], st.full_len[k]), st.half_kind)
            for k in st.p16}


def train_step(st: GPTOracleState, batches, lr=1e-4, betas=(0.9, 0.999), eps=1e-8):
    """One ZeRO-3 step over ``batches`` = [(tokens, targets)] one per rank.

    Returns (mean loss, {key: [fp32 grad shard per rank]}) — the grad shards
    are the reduce-scatter outputs fed to Adam (compared by the parity tests).
    """
    N = st.world
    assert len(batches) == N
    full = gathered(st)
    contribs = {k: [] for k in st.p16}
    losses = []
    for r in range(N):
        loss, g = forward_backward(st.cfg, full, *batches[r])
        losses.append(np.float32(loss))
        for k in st.p16:
            contribs[k].append(nx.round_half(g[k].astype(np.float32), st.half_kind))
    st.step += 1
    cst = AdamConsts.make(lr, betas[0], betas[1], eps, st.step)
    scale = np.float32(1.0 / N)
    gshards = {}
    for k in st.p16:
        shards = reduce_scatter(contribs[k], N, np.float32)
        gshards[k] = []
        for r in range(N):
            g = shards[r] * scale
            gshards[k].append(g)
            P, M, V = adam_update(st.p32[k][r], st.m[k][r], st.v[k][r], g, cst)
            st.p32[k][r], st.m[k][r], st.v[k][r] = P, M, V
            st.p16[k][r] = nx.f32_to_half_bits(P, st.half_kind)
    loss = losses[0]
    for x in losses[1:]:
        loss = np.float32(loss + x)
    return float(loss * scale), gshards
