"""ZeRO-3 / ZeRO-Infinity partitioned training step for a GPT-style model on B200.

The train-harness of SPEC.md:704-799 generalised to the BASELINE GPT
configs. Per operator (embed, each block, head):

  fetch   gather the bf16 bucket from every rank's shard (zi_allgather,
          prefetched one op ahead on a side stream; N=1 + HBM = zero copy)
  compute forward / backward of the block (cuBLAS GEMMs + SDPA attention
          via torch — plain library math; the partitioning, gradient
          reduction and optimizer are libzinf kernels)
  release the gathered slot returns to a 2-slot ring
  reduce  (backward) zi_rs_adam: rank-order fp32 reduce-scatter of the
          per-rank bf16 gradient buckets fused with the bias-corrected
          Adam update of the fp32 master / m / v shard and the RNE bf16
          working copy, in one HBM pass. No global grad-norm clipping
          exists in the SPEC, so Adam runs per bucket inside
          backward as soon as the bucket's last consumer finished.

Layouts (bit-identical to oracle/gpt.py): one PartitionedTensor per op
bucket (block-flattening), ceil(n/N) shard with zero pad;
shards of all buckets live in per-state flat arenas (p16, p32, m, v) with
each bucket's shard 64-element aligned. Init is shard-local and
counter-based (zi_init_uniform), identical to the oracle's generator.
"""

from __future__ import annotations

import os

import math
from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

from . import _lib, kernels
from .comm import LocalComm
from .partition import shard_len
from .schedule import Timeline, plan_prefetch, trace_schedule
from .store import TierKind

LN_EPS = 1e-5
_ALIGN = 64


@dataclass(frozen=True)
class GPTConfig:
    nl: int = 4
    hd: int = 256
    heads: int = 4
    seq: int = 128
    vocab: int = 512
    batch: int = 4  # per-rank micro-batch (sequences)

    @property
    def head_dim(self) -> int:
        return self.hd // self.heads

    @property
    def tokens(self) -> int:
        return self.batch * self.seq


TINY = GPTConfig()
GPT_1P3B = GPTConfig(nl=24, hd=2048, heads=16, seq=1024, vocab=50304, batch=8)
GPT_10B = GPTConfig(nl=50, hd=4096, heads=32, seq=1024, vocab=50304, batch=8)
GPT_70B = GPTConfig(nl=87, hd=8192, heads=64, seq=1024, vocab=50304, batch=4)


def _bound(fan_in: int) -> float:
    return 1.0 / math.sqrt(fan_in)


def layer_params(c: GPTConfig):
    h = c.hd
    ub = ("u", _bound(h))
    return [
        ("ln1_w", (h,), ("c", 1.0)), ("ln1_b", (h,), ("c", 0.0)),
        ("qkv_w", (3 * h, h), ub), ("qkv_b", (3 * h,), ("c", 0.0)),
        ("proj_w", (h, h), ub), ("proj_b", (h,), ("c", 0.0)),
        ("ln2_w", (h,), ("c", 1.0)), ("ln2_b", (h,), ("c", 0.0)),
        ("fc1_w", (4 * h, h), ub), ("fc1_b", (4 * h,), ("c", 0.0)),
        ("fc2_w", (h, 4 * h), ("u", _bound(4 * h))), ("fc2_b", (h,), ("c", 0.0)),
    ]


def embed_params(c: GPTConfig):
    ub = ("u", _bound(c.hd))
    return [("wte", (c.vocab, c.hd), ub), ("wpe", (c.seq, c.hd), ub)]


def final_params(c: GPTConfig):
    return [("lnf_w", (c.hd,), ("c", 1.0)), ("lnf_b", (c.hd,), ("c", 0.0))]


def _numel(shape) -> int:
    return int(math.prod(shape))


def param_count(c: GPTConfig) -> int:
    n = sum(_numel(s) for _, s, _ in embed_params(c) + final_params(c))
    return n + c.nl * sum(_numel(s) for _, s, _ in layer_params(c))


def model_flops_per_step(c: GPTConfig, ranks: int = 1, causal_executed: bool = False) -> float:
    """6 * tokens * params + the attention score / value matmuls, no recompute.

    The attention term is 12 * B * S^2 * hd * nl (QK^T and PV, forward + backward)
    at the dense-equivalent count, the MFU convention (Megatron-LM / PaLM); the
    causal kernels execute half of it (``causal_executed=True`` counts that). The
    paper's 8*tokens*params (efficiency.py:38-45) counts an activation recompute
    this engine does not perform.
    """
    T = c.tokens * ranks
    attn = 12 * c.batch * ranks * c.seq * c.seq * c.hd * c.nl
    if causal_executed:
        attn //= 2
    return 6.0 * T * param_count(c) + attn


@dataclass
class Bucket:
    op: int
    key: str
    params: list
    numel: int
    shard: int            # L = ceil(numel / N)
    arena_off: int        # offset of this bucket's shard inside each state arena
    views: dict = field(default_factory=dict)   # name -> (offset, shape)

    def segments(self):
        off = 0
        for j, (name, shape, init) in enumerate(self.params):
            n = _numel(shape)
            yield name, off, n, self.op * 64 + j, init
            off += n


def _splitmix_key(seed: int, stream: int) -> int:
    M = (1 << 64) - 1

    def mix(z):
        z &= M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    return mix(((seed * 0x9E3779B97F4A7C15) & M) ^ mix(stream + 0x632BE59BD9B4E019))


@dataclass
class Placement:
    """Where model states live (PAPER Table 3)."""
    params: TierKind = TierKind.DEVICE     # bf16 working shards
    optim: TierKind = TierKind.DEVICE      # fp32 master / m / v shards


_GEMM_SITES = ("qkv.fwd", "proj.fwd", "fc1.fwd", "fc2.fwd", "fc2.dW", "fc2.dx", "fc1.dW",
               "fc1.dx", "proj.dW", "proj.dx", "qkv.dW", "qkv.dx", "head.fwd", "head.dW",
               "head.dx")


class GPTZeroEngine:
    """Partitioned ZeRO-3 engine over a communicator (LocalComm or DistComm)."""

    def __init__(self, cfg: GPTConfig, comm=None, seed: int = 7,
                 half_dtype: torch.dtype = torch.bfloat16,
                 compute_dtype: torch.dtype | None = None,
                 placement: Placement | None = None,
                 lr: float = 1e-4, betas=(0.9, 0.999), eps: float = 1e-8,
                 prefetch: bool = True, copy_engine_gather: bool | None = None,
                 trace: bool = False, offload_chunk: int = 16 << 20, fused: bool = True,
                 overlap_opt: bool | None = None, act_ckpt: str | None = None,
                 nvme_root: str | None = None, gemm_select: str | None = None,
                 offload_slots: int | None = None, nvme_direct: bool = False,
                 fwd_state_prefetch_every: int = 2, param_cache: int = 0,
                 prefetch_depths=(3, 2, 1), prefetch_budget: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("GPTZeroEngine needs a CUDA device (no CPU fallback)")
        _lib.load()
        self.cfg = cfg
        self.comm = comm if comm is not None else LocalComm(1)
        self.N = self.comm.world
        self.ranks = list(self.comm.ranks())
        self.seed = seed
        self.half = half_dtype
        self.cdt = compute_dtype or half_dtype
        if self.cdt == torch.bfloat16 and (cfg.seq % 128 or cfg.head_dim not in (64, 128)):
            raise ValueError("bf16 attention (zi_attn) needs seq % 128 == 0 and head_dim 64 or 128")
        self.placement = placement or Placement()
        # bf16 params off HBM: pinned host DRAM, or .shard files on NVMe streamed
        # NVMe -> pinned -> HBM -> gather (the nc / cg / gg stages of PAPER §6.2)
        self.host_params = self.placement.params in (TierKind.HOST, TierKind.NVME)
        self.nvme_params = self.placement.params is TierKind.NVME
        if self.nvme_params and self.placement.optim is not TierKind.HOST:
            raise NotImplementedError("params on NVMe: optimizer states in pinned host DRAM")
        if self.nvme_params and compute_dtype not in (None, half_dtype):
            raise NotImplementedError("params on NVMe: bf16 compute")
        # prefetch plan: while fetch position p runs, issue the nc of
        # p + d_nc, the cg of p + d_cg and the gg of p + d_gg; prefetch_budget (bytes,
        # SPEC.md:621) delays an early nc / cg while the prefetched-but-unconsumed bytes
        # would exceed it (a stage is always issued by the time its successor needs it)
        d_nc, d_cg, d_gg = prefetch_depths
        if not (d_nc >= d_cg >= d_gg >= 1) or d_gg != 1:
            raise ValueError("prefetch depths need d_nc >= d_cg >= d_gg == 1")
        self.depths = tuple(prefetch_depths)
        self.prefetch_budget = prefetch_budget
        self.nvme = self.placement.optim is TierKind.NVME
        if self.nvme and (self.placement.params is not TierKind.DEVICE or not self.comm.is_local):
            raise NotImplementedError("NVMe optimizer states: params in HBM, simulated ranks")
        self.nvme_root = nvme_root
        self.nvme_direct = nvme_direct   # NVMe states through the native O_DIRECT engine
        self.lr, self.betas, self.eps = lr, betas, eps
        self.offload_chunk = offload_chunk
        # staging ring depth (slots of offload_chunk fp32 p/m/v): 24 (4.6 GB at 16 M) with
        # params in HBM; 12 with params on the host, whose own H2D the ring's prefetch
        # would otherwise crowd out during the forward (measured: bench config legs)
        self.offload_slots = offload_slots
        # params on the host: one optimizer-state chunk H2D per this many forward
        # blocks, queued behind their parameter fetches (0: all after the forward)
        self.fwd_state_prefetch_every = fwd_state_prefetch_every
        # reuse distance (ZeRO-3's max_reuse_distance): the forward's last `param_cache`
        # blocks stay gathered in their own HBM slots, and the backward, which starts with
        # them, does not fetch them again (with params on the host: that many fewer
        # parameter H2Ds per step; with peers: fewer NVLink gathers)
        self.param_cache = max(0, int(param_cache))
        # RS + Adam on a side stream, overlapped with the next bucket's backward GEMMs:
        # pays with peers (the RS reads them over NVLink) or host transfers in flight;
        # at N=1 in HBM it measured equal to running them in order (69.4-69.7 ms,
        # scripts/ab_overlap.py), and in order the HBM-bound kernel has the GPU to itself
        if overlap_opt is None:
            env = os.environ.get("ZI_OVERLAP_OPT")
            overlap_opt = (env == "1") if env in ("0", "1") else (
                self.N > 1 or self.placement.optim is not TierKind.DEVICE
                or self.placement.params is not TierKind.DEVICE)
        self.overlap_opt = overlap_opt
        if act_ckpt not in (None, "device", "host"):
            raise ValueError("act_ckpt must be None, 'device' or 'host'")
        self.act_ckpt = act_ckpt
        self.prefetch = prefetch
        # One process per GPU: peer shards are pulled by the copy engines, so the
        # gathers use no SMs and overlap the (all-SM) GEMMs of the op before them
        # (SURVEY §7 hard parts); in-process ranks gather with the SM kernel.
        if copy_engine_gather is None:
            copy_engine_gather = not self.comm.is_local and self.N > 1
        self.copy_engine_gather = copy_engine_gather
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.t = 0
        self.trace = trace
        self._spans, self._t0 = [], None
        self._phase = "forward"
        self._build_buckets()
        self._alloc_state()
        self._init_state()
        self.fwd_seq, self.bwd_seq = trace_schedule(self)
        self.plan = plan_prefetch(self.fwd_seq, self.depths)
        self.gather_stream = torch.cuda.Stream(self.dev)
        self.h2d_stream = torch.cuda.Stream(self.dev)
        self.d2h_stream = torch.cuda.Stream(self.dev)
        self.p16_stream = torch.cuda.Stream(self.dev)   # host params: bf16 write-back lane
        self.p16_ready = {}                              # bucket -> its bf16 write-back landed
        self._alloc_work()
        if not self.comm.is_local and self.N > 1:
            # every barrier channel the step uses (0: step start, 1: cg staging, 2: the
            # optimizer stream) exists and is zeroed on every rank before the first step
            self.comm.open_channels((0, 1, 2))
        self.launches = 0  # libzinf kernel launches issued by step()
        self.adam = kernels.DeviceAdamState(lr, betas, eps, device=self.dev)
        self._graph = None
        # bf16 path: LayerNorm / bias-grad / GELU-bwd / softmax-CE on libzinf kernels
        self.fused = (self.cdt == torch.bfloat16
                      and cfg.hd in (128, 256, 512, 1024, 2048, 4096, 8192)
                      and fused)
        self.ws = kernels.Workspace(max(4 << 20, 2 * 148 * cfg.hd, 600 * 4 * cfg.hd),
                                    device=self.dev) if self.fused else None
        # GEMM epilogue side outputs (fc1 bias colsum, attention delta); ZI_EPI_AUX=0
        # runs the separate passes instead (A/B only)
        self.epi_aux = os.environ.get("ZI_EPI_AUX", "1") != "0"
        # fc2.dx epilogue's 32-row block column sums of du (the fc1 bias gradient)
        self._csum = torch.empty(-(-cfg.tokens // 32) * 4 * cfg.hd if self.fused else 0,
                                 dtype=torch.float32, device=self.dev)
        # Deferred folds: the block backward's four column folds (fc1 / qkv bias, LN2 / LN1
        # gamma, beta and the residual-sum bias) as one zi_fold_sets launch at the end of the
        # block instead of four (the same order, bitwise the same gradients). ZI_FOLD_DEFER=0
        # folds after each producer (A/B only).
        self.fold_defer = self.fused and os.environ.get("ZI_FOLD_DEFER", "1") != "0"
        if self.fold_defer:
            sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
            lnp = 3 * 2 * sms * cfg.hd
            self._csum_qkv = torch.empty(-(-cfg.tokens // 32) * 3 * cfg.hd, dtype=torch.float32,
                                         device=self.dev)
            self._lnpart = [torch.empty(lnp, dtype=torch.float32, device=self.dev) for _ in range(2)]
        # Every linear of the block and the head runs on zi_gemm_sk (tcgen05 stream-K,
        # the neighbouring elementwise pass folded into its epilogue where the site has
        # one): "zi", the default. "cublas" (cuBLAS + a separate pass) and "auto" (time
        # both once per process, keep the faster per site; gemm_select.py) exist for A/B
        # measurements only. ZI_GEMM_SELECT overrides.
        mode = gemm_select or os.environ.get("ZI_GEMM_SELECT", "zi")
        if mode not in ("auto", "zi", "cublas"):
            raise ValueError("gemm_select must be 'auto', 'zi' or 'cublas'")
        self.gemm_select = mode
        self.gsel = {}
        if self.fused:
            if mode == "auto":
                from .gemm_select import tune_gpt
                self.gsel = tune_gpt(cfg.batch * cfg.seq, cfg.hd, cfg.vocab, self.ws, self.dev)
            else:
                self.gsel = dict.fromkeys(_GEMM_SITES, mode)

    # ------------------------------------------------------------------ layout
    def _build_buckets(self):
        c = self.cfg
        specs = [(0, "embed", embed_params(c))]
        specs += [(i + 1, f"h{i}", layer_params(c)) for i in range(c.nl)]
        specs.append((c.nl + 1, "final", final_params(c)))
        self.buckets: list[Bucket] = []
        off = 0
        for op, key, params in specs:
            n = sum(_numel(s) for _, s, _ in params)
            L = shard_len(n, self.N)
            b = Bucket(op, key, params, n, L, off)
            o = 0
            for name, shape, _ in params:
                b.views[name] = (o, shape)
                o += _numel(shape)
            self.buckets.append(b)
            off += -(-L // _ALIGN) * _ALIGN
        self.arena_len = off
        self.by_key = {b.key: b for b in self.buckets}

    def operators(self):
        """[(param keys, bytes, flops)] in forward order, for trace_schedule."""
        c = self.cfg
        out = []
        for b in self.buckets:
            keys = (b.key,) if b.key != "final" else ("final", "embed")  # tied wte (external)
            flops = 2 * c.tokens * b.numel if b.key != "embed" else c.tokens * c.hd
            if b.key == "final":
                flops += 2 * c.tokens * c.vocab * c.hd
            out.append((keys, 2 * b.numel, max(1, flops)))
        return out

    def _alloc_state(self):
        nloc = len(self.ranks)
        A = self.arena_len
        hp = self.host_params
        ho = self.placement.optim is TierKind.HOST

        self._pinned = []

        def mk(dtype, host):
            if host:  # exact-size cudaHostAlloc (zi_host_alloc): copy-engine DMA source/target
                from .store import _PinnedBuffer
                nbytes = nloc * A * torch.empty(0, dtype=dtype).element_size()
                buf = _PinnedBuffer(nbytes)
                self._pinned.append(buf)
                t = buf.tensor.view(dtype).view(nloc, A)
                t.zero_()
                return t
            return torch.zeros(nloc, A, dtype=dtype, device=self.dev)
        if hp or self.comm.is_local:
            self.p16 = mk(self.half, hp)
        else:  # peers gather from it over NVLink: an IPC-shareable allocation
            self.p16 = self.comm.alloc((nloc, A), self.half)
        if self.nvme_params:
            # bf16 param shards live in reference-format .shard files ({bucket}.p16/rank{r});
            # the pinned arena above is the write-back staging the updates land in
            import tempfile
            from concurrent.futures import ThreadPoolExecutor
            from .store import TierStore
            root = self.nvme_root or tempfile.mkdtemp(prefix="zinf-nvme-params-")
            self.pstore = TierStore(0, 0, nvme_root=root, workers=8)
            self._io = ThreadPoolExecutor(max_workers=8, thread_name_prefix="zinf-nc")
        if self.nvme:  # optimizer states live in .shard files (nvme_opt.NvmeOptimizerStreamer)
            import tempfile
            from .nvme_opt import NvmeOptimizerStreamer
            from .store import TierStore
            root = self.nvme_root or tempfile.mkdtemp(prefix="zinf-nvme-")
            self.store = TierStore(0, 0, nvme_root=root, workers=8)
            self.streamer = NvmeOptimizerStreamer(self, self.store, direct=self.nvme_direct)
            self.p32 = self.m = self.v = None
            return
        self.p32 = mk(torch.float32, ho)
        self.m = mk(torch.float32, ho)
        self.v = mk(torch.float32, ho)

    def _init_state(self):
        """Shard-local counter-RNG init; never a full tensor."""
        ho = self.placement.optim is TierKind.HOST
        hp = self.host_params
        for li, r in enumerate(self.ranks):
            for b in self.buckets:
                lo, hi = r * b.shard, min((r + 1) * b.shard, b.numel)
                if hi <= lo:
                    continue
                # stage on device when the tiers are host / NVMe, then copy down
                p32 = torch.zeros(b.shard, dtype=torch.float32, device=self.dev) \
                    if (ho or self.nvme) else self.p32[li, b.arena_off:b.arena_off + b.shard]
                p16 = torch.empty(b.shard, dtype=self.half, device=self.dev) if hp else \
                    self.p16[li, b.arena_off:b.arena_off + b.shard]
                for name, off, n, stream, init in b.segments():
                    s, e = max(lo, off), min(hi, off + n)
                    if s >= e:
                        continue
                    d32 = p32[s - lo:e - lo]
                    d16 = p16[s - lo:e - lo]
                    if init[0] == "u":
                        kernels.init_uniform(d32, d16, _splitmix_key(self.seed, stream), s - off,
                                             float(init[1] * 2.0 ** -24))
                    else:
                        kernels.fill(d32, d16, float(init[1]))
                if ho:
                    self.p32[li, b.arena_off:b.arena_off + b.shard].copy_(p32)
                if self.nvme:
                    torch.cuda.synchronize()
                    self.streamer.put_initial(b.key, r, p32)
                if hp:
                    self.p16[li, b.arena_off:b.arena_off + b.shard].copy_(p16)
        torch.cuda.synchronize()
        if self.nvme_params:   # the initial bf16 shards become the param files
            tickets = [self.pstore.write(self._pkey(b, r),
                                         self.p16[li, b.arena_off:b.arena_off + b.shard],
                                         TierKind.NVME)
                       for li, r in enumerate(self.ranks) for b in self.buckets]
            self.pstore.flush(tickets)

    def _alloc_work(self):
        c = self.cfg
        maxn = max(b.shard * self.N for b in self.buckets if b.key != "embed")
        e = self.by_key["embed"]
        # gathered-parameter slots: a 2-slot ring for blocks/final + a resident embed slot
        self.zero_copy = self.N == 1 and self.placement.params is TierKind.DEVICE and self.cdt == self.half
        nb = len(self.buckets) - 2
        self.K = min(self.param_cache, max(0, nb - 1)) if not self.zero_copy else 0
        if not self.zero_copy:   # 2-slot ring + K reuse-cache slots
            self.slots = [torch.empty(maxn, dtype=self.half, device=self.dev)
                          for _ in range(2 + self.K)]
            self.embed_slot = torch.empty(e.shard * self.N, dtype=self.half, device=self.dev)
        if self.cdt != self.half:
            self.wide_slots = [torch.empty(maxn, dtype=self.cdt, device=self.dev)
                               for _ in range(2 + getattr(self, "K", 0))]
            self.wide_embed = torch.empty(e.shard * self.N, dtype=self.cdt, device=self.dev)
        self.slot_ready = [None, None]
        # gradient contribution buckets: per local rank, 2-slot ring + embed slot
        nloc = len(self.ranks)
        sh = self.comm.alloc  # IPC-shareable when peers read the contributions
        self.gslots = [[sh((maxn,), self.half) for _ in range(2)]
                       for _ in range(nloc)]
        self.gembed = [sh((e.shard * self.N,), self.half) for _ in range(nloc)]
        if self.cdt != self.half:
            self.gwide = [torch.zeros(maxn, dtype=self.cdt, device=self.dev) for _ in range(nloc)]
        self.wte_acc = [torch.zeros(c.vocab, c.hd, dtype=torch.float32, device=self.dev)
                        for _ in range(nloc)]
        self.emb_work = torch.empty(2 * c.vocab + 1 + c.tokens, dtype=torch.int32, device=self.dev)
        if not self.comm.is_local and self.N > 1:
            self.peer_gslots = [self.comm.share(self.gslots[0][k]) for k in range(2)]
            self.peer_gembed = self.comm.share(self.gembed[0])
            if self.host_params:
                # cg staging slots (embed + 2-slot ring) that peers gather from
                shmax = max(b.shard for b in self.buckets)
                self.pstage = [self.comm.alloc((shmax,), self.half) for _ in range(3)]
                self.peer_pstage = [self.comm.share(s) for s in self.pstage]
            else:
                self.peer_p16 = self.comm.share(self.p16[0])
        self.events = {}
        # staged fetch (params off HBM): cg staging slots in HBM (simulated ranks; with
        # peers the IPC pstage ring plays that part) and, for NVMe params, pinned nc slots
        # that the store workers read the shard files into
        self._flist = self._fetch_list()
        self._fplan = None
        self.issue_log, self.nc_bytes = [], 0
        self._staged, self._cg_ev, self._cg_free, self._cg_issued = {}, {}, {}, set()
        self._nc_fut, self._nc_busy, self._nc_issued = {}, {}, set()
        self._p16_wfut = {}
        self._fpos = 0
        if self.host_params:
            shmax = max(b.shard for b in self.buckets)
            self.CGS = self.depths[1] + 1
            if self.comm.is_local:
                self.cg_slots = [[torch.empty(shmax, dtype=self.half, device=self.dev)
                                  for _ in range(nloc)] for _ in range(self.CGS)]
            if self.nvme_params:
                from .store import _PinnedBuffer
                self.NCS = self.depths[0] + 1
                per = shmax * torch.empty(0, dtype=self.half).element_size()
                self._nc_buf = _PinnedBuffer(self.NCS * nloc * per)
                flat = self._nc_buf.tensor.view(self.half)
                self.nc_slots = [[flat[(k * nloc + li) * shmax:(k * nloc + li + 1) * shmax]
                                  for li in range(nloc)] for k in range(self.NCS)]
        # offload engine: double-buffered HBM staging for optimizer-state chunks
        self.offload = self.placement.optim is TierKind.HOST
        self.opt_stream = torch.cuda.Stream(self.dev)
        self._pending_free = None
        # activation checkpoints: block inputs in pinned host DRAM + a 2-slot HBM ring
        self._ckpt_saved, self._ckpt_loaded, self.ckpt_bytes = {}, {}, 0
        if self.act_ckpt == "host":
            from .store import _PinnedBuffer
            per = c.tokens * c.hd
            self._ckpt_buf = _PinnedBuffer(nloc * c.nl * per * 2)
            flat = self._ckpt_buf.tensor.view(torch.bfloat16)
            self.ckpt_host = [[flat[(li * c.nl + i) * per:(li * c.nl + i + 1) * per]
                               for i in range(c.nl)] for li in range(nloc)]
            self.ckpt_ring = [[torch.empty(c.tokens, c.hd, dtype=torch.bfloat16, device=self.dev)
                               for _ in range(2)] for _ in range(nloc)]
        self.gfree = {}          # grad slot -> event: optimizer finished reading it
        if self.offload:
            # The step's optimizer-state chunks in the order the backward consumes them
            # (head bucket, blocks last-to-first, embed), every local rank's shard in
            # balanced chunks. They stream through a ring of NS HBM staging slots:
            # chunk q lives in slot (base + q) % NS, its H2D is issued NS-1 chunks
            # ahead of its rs_adam and waits only for the D2H that last drained the slot.
            C = self.offload_chunk
            self._ochunks, self._obucket = [], {}
            order = [self.buckets[-1]] + self.buckets[1:-1][::-1] + [self.buckets[0]]
            for b in order:
                idx = []
                for li in range(nloc):
                    L = b.shard
                    nch = -(-L // C)
                    cs = -(-L // nch)                 # balanced chunks, no runt tail
                    for s0 in range(0, L, cs):
                        idx.append(len(self._ochunks))
                        self._ochunks.append((b, li, s0, min(cs, L - s0)))
                self._obucket[b.key] = idx
            # NS <= chunks per step: the in-order D2H stream then guarantees that chunk
            # q's previous-step write-back landed before its next H2D (slot reuse events)
            want = self.offload_slots or (12 if self.host_params else 24)
            NS = max(3, min(want, len(self._ochunks)))
            self.stage = [[torch.empty(C, dtype=torch.float32, device=self.dev) for _ in range(3)]
                          for _ in range(NS)]
            self.stage16 = [torch.empty(C, dtype=self.half, device=self.dev) for _ in range(NS)]
            self.ev_d2h = [None] * NS
            self._obase = 0          # global index of this step's chunk 0
            self._oh2d = {}          # chunk -> H2D-complete event (this step)
            self.offload_bytes = 0

    # ------------------------------------------------------------- fetch/release
    def _shard_view(self, arena, li, b: Bucket):
        return arena[li, b.arena_off:b.arena_off + b.shard]

    # ------------------------------------------------------------------ tracing
    def _tmark(self, stream):
        """Timing event on `stream` (only while tracing)."""
        if not self.trace:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def _tspan(self, op: int, stage: str, e0, e1) -> None:
        if e0 is not None and e1 is not None:
            self._spans.append((op, stage, e0, e1, self._phase))

    def timeline(self, phase: str | None = None) -> Timeline:
        """Timeline of the last traced step, seconds from step start.

        ``phase`` = "forward" | "backward" keeps only that pass's spans (the
        head's fused forward + backward counts as the first backward op).
        """
        torch.cuda.synchronize()
        tl = Timeline(t0=0.0)
        for op, stage, e0, e1, ph in self._spans:
            if phase is None or ph == phase:
                tl.add(op, stage, self._t0.elapsed_time(e0) / 1e3, self._t0.elapsed_time(e1) / 1e3)
        return tl

    def simulated_step(self, duplex: bool = False, lanes: dict | None = None) -> dict:
        """Replay the last traced step's measured per-op stage costs through the lane simulator.

        This is the calibration of SURVEY §8 f4. ``costs_from_timeline`` takes
        each op's measured stage durations. ``simulate`` / ``simulate_backward``
        schedule them with the engine's plan: one-op-ahead fetches, so depths
        (1, 1, 1); the head is the first backward op and the embedding the
        last. Comparing with the measured step tests the simulator's lane model.

        In the offload placement a bucket's optimizer-state H2D is its ``cg``
        stage, prefetched through the staging ring: the ring runs NS-1 chunks
        ahead, i.e. ``d`` ops at the block buckets' chunk count, so the backward
        plan has depths (d, d, 1). Its D2H is the post-compute ``grad_offload``.
        With ``duplex=False`` both share the SPEC's single ``pcie`` lane; with
        ``duplex=True`` they run on ``pcie_h2d`` / ``pcie_d2h``, the two copy
        engines of a full-duplex link. The simulator runs the forward and the
        backward back to back, so the ring's prefetch during the forward and the
        write-back drained into the next forward are outside its model.
        """
        from .schedule import (Op, OperatorSequence, costs_from_timeline, plan_prefetch,
                               simulate, simulate_backward)
        E, FB, blocks = self.buckets[0], self.buckets[-1], self.buckets[1:-1]
        fwd_ops = [E.op] + [b.op for b in blocks]
        bwd_ops = [FB.op] + [b.op for b in reversed(blocks)] + [E.op]

        def plan(ids, depths=(1, 1, 1)):
            return plan_prefetch(OperatorSequence(tuple(Op(i, (), 1, 1) for i in ids),
                                                 "backward"), depths)
        fwd_tl, bwd_tl = self.timeline("forward"), self.timeline("backward")
        bwd_depths = (1, 1, 1)
        if self.offload:
            per_op = len(self._obucket[(blocks[0] if blocks else FB).key])
            d = max(1, -(-(len(self.stage) - 1) // max(1, per_op)))
            bwd_depths = (d, d, 1)
        if duplex:
            lanes = dict({"cg": "pcie_h2d", "grad_offload": "pcie_d2h"}, **(lanes or {}))
        fc = costs_from_timeline(fwd_tl, fwd_ops)
        bc = costs_from_timeline(bwd_tl, bwd_ops)
        sf = simulate(plan(fwd_ops), fc, lanes=lanes)
        sb = simulate_backward(plan(bwd_ops, bwd_depths), bc, lanes=lanes)
        measured = self.timeline().total_s
        predicted = sf.total_s + sb.total_s
        return {"measured_s": measured, "predicted_s": predicted,
                "rel_error": (predicted - measured) / measured if measured else 0.0,
                "forward_predicted_s": sf.total_s, "backward_predicted_s": sb.total_s,
                "serial_s": sf.serial_s + sb.serial_s, "forward": sf, "backward": sb}

    def _fetch(self, b: Bucket, slot: int, stream):
        """The gg stage of the step's next fetch position p: gather bucket b into
        gathered slot `slot` on `stream`. It first issues what the prefetch plan
        schedules while position p - 1 runs (the nc of p - 1 + d_nc, the cg of
        p - 1 + d_cg) and whatever p itself still lacks."""
        if self.zero_copy:
            return
        p = self._fpos
        self._fpos += 1
        self._advance(p)
        staged = self.comm.is_local and self.host_params   # gg reads the cg staging slot
        dst = self.embed_slot if b.key == "embed" else self.slots[slot]
        with torch.cuda.stream(stream):
            t0 = self._tmark(stream)
            if self.host_params:   # cg bytes over the host link
                self.fetch_bytes = getattr(self, "fetch_bytes", 0) + b.shard * len(self.ranks) * 2
            if staged:
                stream.wait_event(self._cg_ev.pop(p))
                k = p % self.CGS
                shards = [self.cg_slots[k][li][:b.shard] for li in range(len(self.ranks))]
                kernels.allgather(shards, b.shard, dst, b.numel,
                                  use_copy_engine=self.copy_engine_gather)
            elif self.comm.is_local:
                shards = [self._shard_view(self.p16, li, b) for li in range(len(self.ranks))]
                kernels.allgather(shards, b.shard, dst, b.numel,
                                  use_copy_engine=self.copy_engine_gather)
            elif self.host_params:
                # source of our shard: the pinned arena, or the nc slot the NVMe read filled
                if self.nvme_params:
                    for f in self._nc_fut.pop(p):
                        f.result()
                    src = self.nc_slots[p % self.NCS][0][:b.shard]
                else:
                    ev = self.p16_ready.pop(b.key, None)
                    if ev is not None:   # the previous step's bf16 shard is back in host DRAM
                        stream.wait_event(ev)
                    src = self._shard_view(self.p16, 0, b)
                # ZeRO-Infinity fetch (PAPER §6.2): cg = H2D of our pinned shard into an
                # IPC-shared HBM staging slot, then gg = P2P gather of every rank's slot.
                # The gather-channel barrier before the gg makes all ranks' cg visible; the
                # next fetch's barrier keeps a slot from being refilled while peers read it.
                # the two ring stages alternate per fetch (not per slot: the backward
                # skips the re-fetch of the last block, so slots do not alternate there)
                if b.key == "embed":
                    k = 0
                else:
                    self._pstage_n = getattr(self, "_pstage_n", 0) + 1
                    k = 1 + self._pstage_n % 2
                stage = self.pstage[k]
                stage[:b.shard].copy_(src, non_blocking=True)
                if self.nvme_params:   # the nc slot is free once this H2D has read it
                    evb = torch.cuda.Event()
                    evb.record(stream)
                    self._nc_busy[p % self.NCS] = evb
                self.comm.device_barrier(stream, channel=1)
                kernels.allgather(self.peer_pstage[k], b.shard, dst, b.numel,
                                  use_copy_engine=self.copy_engine_gather)
            else:
                base = b.arena_off * self.p16.element_size()
                ptrs = [p + base for p in self.peer_p16]
                kernels.allgather(ptrs, b.shard, dst, b.numel,
                                  use_copy_engine=self.copy_engine_gather)
            if self.cdt != self.half:
                wide = self.wide_embed if b.key == "embed" else self.wide_slots[slot]
                kernels.cast_half_to_f32(dst[:b.numel], wide[:b.numel])
            self._tspan(b.op, "cg" if (self.host_params and not staged) else "gg",
                        t0, self._tmark(stream))
            ev = torch.cuda.Event()
            ev.record(stream)
        if staged:   # the cg slot may be refilled once this gather has read it
            self._cg_free[p % self.CGS] = ev
        self._staged.pop(p, None)
        self.events[(b.key, slot)] = ev

    # ----------------------------------------------- staged fetch: nc / cg (PAPER §6.2)
    def _fetch_list(self) -> list:
        """The step's fetch positions in the order ``_fetch`` runs them: embed, the
        blocks and the head (forward), then the blocks the backward gathers again (all
        but the last one and the K reuse-cached ones, last to first)."""
        blocks, E, FB = self.buckets[1:-1], self.buckets[0], self.buckets[-1]
        nb = len(blocks)
        back = [blocks[j] for j in range(nb - 2 - self.K, -1, -1)]
        return [E] + blocks + [FB] + back

    def _budget_ok(self, q: int) -> bool:
        if self.prefetch_budget is None:
            return True
        need = self._flist[q].shard * len(self.ranks) * 2
        return sum(self._staged.values()) + need <= self.prefetch_budget

    def _advance(self, p: int) -> None:
        """Issue the plan's nc / cg stages for fetch position p: the
        eager set at p == 0, ``plan.issue(p - 1)`` otherwise, within the byte budget —
        after p's own nc and cg if they are still missing (the copy FIFOs serve p first)."""
        if not self.host_params:
            return
        self._nc(p, p, forced=True)
        self._cg(p, p, forced=True)
        todo = self._fplan.slots[0] if p == 0 else self._fplan.issue(p - 1)
        for q in todo["nc"]:
            self._nc(q, p, forced=False)
        for q in todo["cg"]:
            self._cg(q, p, forced=False)

    def _nc(self, q: int, at: int, forced: bool) -> None:
        """nc-transfer of fetch position q: every local rank's bf16 shard file is read
        by a store worker into pinned nc slot q % NCS (after the slot's previous H2D
        has read it, and after the file's last write-back)."""
        if not self.nvme_params or q >= len(self._flist) or q in self._nc_issued:
            return
        if not forced and not self._budget_ok(q):
            return
        b = self._flist[q]
        k = q % self.NCS
        busy = self._nc_busy.pop(k, None)
        futs = []
        for li, r in enumerate(self.ranks):
            view = self.nc_slots[k][li][:b.shard]
            futs.append(self._io.submit(self._nc_job, self._pkey(b, r), view,
                                        self._p16_wfut.get((b.key, r)), busy))
        self._nc_fut[q] = futs
        self._nc_issued.add(q)
        self._staged[q] = b.shard * len(self.ranks) * 2
        self.issue_log.append((at, "nc", q))
        self.nc_bytes += b.shard * len(self.ranks) * 2

    def _nc_job(self, key: str, view: torch.Tensor, wfut, busy) -> None:
        if wfut is not None:
            wfut.result()          # the file holds the last update (read after write)
        if busy is not None:
            busy.synchronize()     # the slot's previous H2D has read it
        self.pstore.read_into(key, TierKind.NVME, view).wait()

    def _wb_job(self, key: str, view: torch.Tensor, ev) -> None:
        ev.synchronize()           # the updated bf16 shard landed in pinned memory
        self.pstore.write_range(key, TierKind.NVME, 0, view).wait()

    def _pkey(self, b: Bucket, r: int) -> str:
        return f"{b.key}.p16/rank{r}"

    def _cg(self, q: int, at: int, forced: bool) -> None:
        """cg-transfer of fetch position q (simulated ranks): every local rank's shard,
        from the pinned arena (HOST) or its nc slot (NVMe), H2D into cg staging slot
        q % CGS, behind the gather that last read the slot."""
        if not (self.comm.is_local and self.host_params) or q >= len(self._flist):
            return
        if q in self._cg_issued:
            return
        if not forced and not self._budget_ok(q):
            return
        b = self._flist[q]
        k = q % self.CGS
        h2d = self.h2d_stream
        if self.nvme_params:
            self._nc(q, at, forced=True)
            for f in self._nc_fut.pop(q):
                f.result()
        with torch.cuda.stream(h2d):
            ev_free = self._cg_free.pop(k, None)
            if ev_free is not None:
                h2d.wait_event(ev_free)
            if self.nvme_params:
                src = [self.nc_slots[q % self.NCS][li][:b.shard] for li in range(len(self.ranks))]
            else:
                evp = self.p16_ready.pop(b.key, None)
                if evp is not None:   # the previous step's bf16 shard is back in host DRAM
                    h2d.wait_event(evp)
                src = [self._shard_view(self.p16, li, b) for li in range(len(self.ranks))]
            t0 = self._tmark(h2d)
            for li in range(len(self.ranks)):
                self.cg_slots[k][li][:b.shard].copy_(src[li], non_blocking=True)
            self._tspan(b.op, "cg", t0, self._tmark(h2d))
            ev = torch.cuda.Event()
            ev.record(h2d)
        self._cg_ev[q] = ev
        self._cg_issued.add(q)
        if self.nvme_params:
            self._nc_busy[q % self.NCS] = ev
        self._staged[q] = b.shard * len(self.ranks) * 2
        self.issue_log.append((at, "cg", q))

    def _pslot(self, i: int, nb: int) -> int:
        """Gathered-parameter slot of block i (i == nb: the head bucket): the last K
        blocks own reuse-cache slots 2.., the others alternate in the 2-slot ring; the
        head takes the ring slot the block before it (or the first cached block) would
        have used, which never holds a block the backward still needs."""
        K = self.K
        if K and i < nb and i >= nb - K:
            return 2 + i - (nb - K)
        return (nb - K) % 2 if (K and i == nb) else i % 2

    def _full(self, b: Bucket, slot: int) -> torch.Tensor:
        """The gathered (compute-dtype) flat bucket, after waiting for its fetch."""
        if self.zero_copy:
            return self.p16[0, b.arena_off:b.arena_off + b.numel]
        ev = self.events.pop((b.key, slot), None)
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)
        if self.cdt != self.half:
            w = self.wide_embed if b.key == "embed" else self.wide_slots[slot]
            return w[:b.numel]
        src = self.embed_slot if b.key == "embed" else self.slots[slot]
        return src[:b.numel]

    def _params(self, b: Bucket, flat: torch.Tensor) -> dict:
        return {n: flat[o:o + _numel(s)].view(s) for n, (o, s) in b.views.items()}

    # ------------------------------------------------------------------ compute
    def _embed_fwd(self, P, tokens):
        c = self.cfg
        if self.fused:   # one libzinf pass: token row + position row, rounded once
            x = torch.empty(tokens.numel(), c.hd, dtype=P["wte"].dtype, device=self.dev)
            kernels.embed_fwd(tokens.contiguous(), P["wte"], P["wpe"][: tokens.shape[1]], x)
            return x
        x = F.embedding(tokens, P["wte"]) + P["wpe"][: tokens.shape[1]]
        return x.reshape(-1, c.hd)

    def _attn_fwd(self, qkv):
        """Causal attention of the block. bf16: libzinf's tcgen05 kernels (zi_attn_fwd; the
        backward is fixed-order, so the step is bitwise reproducible). fp32 / fp16
        compute (the SPEC-parity modes): the same math through torch's SDPA in that dtype."""
        c = self.cfg
        B, S, H, D = c.batch, c.seq, c.heads, c.head_dim
        if self.cdt == torch.bfloat16:
            o = torch.empty(B * S, c.hd, dtype=qkv.dtype, device=qkv.device)
            lse = torch.empty(B * H * S, dtype=torch.float32, device=qkv.device)
            kernels.attn_fwd(qkv, o, lse, B, H)
            return o, (qkv, o, lse)
        leaf = qkv.detach().requires_grad_(True)
        with torch.enable_grad():
            q, k, v = leaf.view(B, S, 3, H, D).unbind(2)
            o4 = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2),
                                                v.transpose(1, 2), is_causal=True)
        o = o4.detach().transpose(1, 2).reshape(B * S, c.hd)
        return o, (leaf, o4)

    def _attn_bwd(self, do, saved, delta=None, colsum=None):
        """delta given: rowsum(do o o) was formed by the GEMM that produced do. colsum: fp32
        [T/32, 3*hd] receiving dqkv's 32-row block column sums (the qkv bias gradient)."""
        c = self.cfg
        if self.cdt == torch.bfloat16:
            qkv, o, lse = saved
            dqkv = torch.empty_like(qkv)
            given = delta is not None
            if not given:
                delta = torch.empty_like(lse)
            kernels.attn_bwd(qkv, None if given else o, do, lse, delta, dqkv, c.batch, c.heads,
                             colsum=colsum)
            return dqkv
        leaf, o4 = saved
        g4 = do.view(c.batch, c.seq, c.heads, c.head_dim).transpose(1, 2)
        (dqkv,) = torch.autograd.grad(o4, leaf, g4)
        return dqkv.reshape(-1, 3 * c.hd)

    def _gelu_save(self) -> bool:
        """fc1's forward epilogue stores GELU'(u) in place of u for fc2's input-gradient
        epilogue (both sites on zi_gemm_sk, side outputs on)."""
        return (self.epi_aux and self.gsel.get("fc1.fwd") == "zi"
                and self.gsel.get("fc2.dx") == "zi")

    def _colsum_part(self, T: int, N: int) -> torch.Tensor:
        """fp32 [ceil(T/32), N] block column sums of a GEMM epilogue (one buffer, reused
        in stream order)."""
        n = -(-T // 32) * N
        if self._csum.numel() < n:
            raise ValueError(f"colsum buffer holds {self._csum.numel()} < {n} floats")
        return self._csum[:n]

    def _ln(self, x, w, b, resid=None):
        """libzinf LayerNorm (bf16); with resid the residual add is fused: returns
        (x + resid, y, mean, rstd)."""
        T = x.shape[0]
        y = torch.empty_like(x)
        mean = torch.empty(T, dtype=torch.float32, device=x.device)
        rstd = torch.empty(T, dtype=torch.float32, device=x.device)
        xs = torch.empty_like(x) if resid is not None else None
        kernels.ln_fwd(x, w, b, y, mean, rstd, LN_EPS, resid=resid, xsum=xs)
        return xs, y, mean, rstd

    def _block_fwd(self, x, P):
        if self.fused:
            return self._block_fwd_fused(x, P)
        hd = self.cfg.hd
        h1, m1, r1 = torch.native_layer_norm(x, (hd,), P["ln1_w"], P["ln1_b"], LN_EPS)
        qkv = torch.addmm(P["qkv_b"], h1, P["qkv_w"].t())
        o, att = self._attn_fwd(qkv)
        x2 = torch.addmm(P["proj_b"], o, P["proj_w"].t())
        x2 += x
        h2, m2, r2 = torch.native_layer_norm(x2, (hd,), P["ln2_w"], P["ln2_b"], LN_EPS)
        u = torch.addmm(P["fc1_b"], h2, P["fc1_w"].t())
        a = F.gelu(u, approximate="tanh")
        y = torch.addmm(P["fc2_b"], a, P["fc2_w"].t())
        y += x2
        return y, (x, h1, m1, r1, att, o, x2, h2, m2, r2, u, a)

    def _zi(self, site: str, *ts) -> bool:
        """Run ``site`` on zi_gemm_sk (the product path); its operands must meet the
        kernel's alignment contract — no silent library fallback."""
        if self.gsel.get(site) != "zi":
            return False
        from .gemm_select import aligned
        if not aligned(*ts):
            raise ValueError(f"{site}: operands not 16-byte aligned for zi_gemm_sk")
        return True

    def _linear(self, site, x, w, b, out=None):
        """y = x w^T + b on the site's chosen GEMM."""
        if out is None:
            out = torch.empty(x.shape[0], w.shape[0], dtype=x.dtype, device=x.device)
        if self._zi(site, x, w, b, out):
            kernels.gemm_sk(x, w, out, bias=b)
        else:
            torch.addmm(b, x, w.t(), out=out)
        return out

    def _mm_dw(self, site, dy, inp, out):
        """out = dy^T inp (a weight gradient, written into its grad-bucket view)."""
        if self._zi(site, dy, inp, out):
            kernels.gemm_sk(dy.t(), inp.t(), out)
        elif out.dtype == dy.dtype:
            torch.mm(dy.t(), inp, out=out)
        else:
            torch.ops.aten.mm.dtype_out(dy.t(), inp, out.dtype, out=out)  # fp32 out, no copy
        return out

    def _mm_dx(self, site, dy, w):
        """dy w (an input gradient)."""
        out = torch.empty(dy.shape[0], w.shape[1], dtype=dy.dtype, device=dy.device)
        if self._zi(site, dy, w, out):
            kernels.gemm_sk(dy, w.t(), out)
        else:
            torch.mm(dy, w, out=out)
        return out

    def _block_fwd_fused(self, x, P):
        """bf16 block with libzinf LayerNorms; the attention residual add is fused
        into LN2 (x2 = x + proj(o), h2 = LN(x2) in one pass). Each linear runs on
        its site's GEMM (zi_gemm with bias / GELU / residual epilogues, or cuBLAS +
        the separate pass)."""
        _, h1, m1, r1 = self._ln(x, P["ln1_w"], P["ln1_b"])
        qkv = self._linear("qkv.fwd", h1, P["qkv_w"], P["qkv_b"])
        o, att = self._attn_fwd(qkv)
        p = self._linear("proj.fwd", o, P["proj_w"], P["proj_b"])
        x2, h2, m2, r2 = self._ln(p, P["ln2_w"], P["ln2_b"], resid=x)
        del p
        T, H4 = h2.shape[0], P["fc1_w"].shape[0]
        u = torch.empty(T, H4, dtype=h2.dtype, device=h2.device)
        a = torch.empty_like(u)
        if self._zi("fc1.fwd", h2, P["fc1_w"], P["fc1_b"], u, a):
            # with the GELU'-saving epilogue, "u" holds GELU'(u): the fc2 input-gradient
            # GEMM then only multiplies (its epilogue no longer evaluates tanh)
            kernels.gemm_sk(h2, P["fc1_w"], u, bias=P["fc1_b"],
                            epi="gelu_save" if self._gelu_save() else "gelu", out2=a)
        else:
            torch.addmm(P["fc1_b"], h2, P["fc1_w"].t(), out=u)
            kernels.gelu_fwd(u, a)
        y = torch.empty_like(x2)
        if self._zi("fc2.fwd", a, P["fc2_w"], P["fc2_b"], y, x2):
            kernels.gemm_sk(a, P["fc2_w"], y, bias=P["fc2_b"], epi="resid", x=x2)
        else:
            torch.addmm(P["fc2_b"], a, P["fc2_w"].t(), out=y)
            y += x2
        return y, (x, h1, m1, r1, att, o, x2, h2, m2, r2, u, a)

    def _block_bwd_fused(self, dy, cache, P, G):
        """bf16 block backward: bias grads via deterministic column sums, GELU
        backward fused with the fc1 bias grad (or into the fc2 input-gradient GEMM's
        epilogue), LayerNorm backward with the residual gradient folded in — all
        libzinf; GEMMs on zi_gemm_sk, attention on zi_attn (tcgen05)."""
        x, h1, m1, r1, att, o, x2, h2, m2, r2, u, a = cache
        ws = self.ws
        folds = []     # (part, P, N, out) sets folded in one launch at the end (fold_defer)
        self._mm_dw("fc2.dW", dy, a, G["fc2_w"])
        du = torch.empty_like(u)
        if self._zi("fc2.dx", dy, P["fc2_w"], du, u) and self.epi_aux:
            # du = (dy W2) * gelu'(u); the epilogue also sums du's columns per 32-row
            # block, so db1 is one small fold instead of a pass over du
            T, H4 = du.shape
            part = self._colsum_part(T, H4)
            kernels.gemm_sk(dy, P["fc2_w"].t(), du, epi="mul" if self._gelu_save() else "dgelu",
                            x=u, colsum=part)
            if self.fold_defer:
                folds.append((part, -(-T // 32), H4, G["fc1_b"]))
            else:
                kernels.colsum_fold(part, -(-T // 32), H4, G["fc1_b"])
        elif self._zi("fc2.dx", dy, P["fc2_w"], du, u):   # A/B: separate bias pass
            kernels.gemm_sk(dy, P["fc2_w"].t(), du, epi="dgelu", x=u)
            kernels.bias_grad(du, G["fc1_b"], ws)
        else:
            da = torch.mm(dy, P["fc2_w"])
            kernels.bias_grad(da, G["fc1_b"], ws, u=u, du=du)
            del da
        self._mm_dw("fc1.dW", du, h2, G["fc1_w"])
        dh2 = self._mm_dx("fc1.dx", du, P["fc1_w"])
        del du
        dx2 = torch.empty_like(dh2)
        # LN2 backward also sums dres = dy: the fc2 bias gradient, no extra pass
        self._ln_bwd_fold(folds, 0, dh2, x2, P["ln2_w"], m2, r2, dx2, G["ln2_w"], G["ln2_b"],
                          dres=dy, dres_sum=G["fc2_b"])
        self._mm_dw("proj.dW", dx2, o, G["proj_w"])
        if self._zi("proj.dx", dx2, P["proj_w"], o) and self.epi_aux:
            # dO = dx2 Wp; the epilogue also forms the attention backward's
            # delta = rowsum(dO o O) per head, so zi_attn_bwd skips its delta pass
            c = self.cfg
            do = torch.empty(dx2.shape[0], P["proj_w"].shape[1], dtype=dx2.dtype, device=dx2.device)
            delta = torch.empty(c.batch * c.heads * c.seq, dtype=torch.float32, device=dx2.device)
            kernels.gemm_sk(dx2, P["proj_w"].t(), do, x=o, delta=delta,
                            delta_shape=(c.seq, c.heads, c.head_dim))
            # the attention backward's epilogues also sum dqkv's columns per 32-row block:
            # the qkv bias gradient is one small fold instead of a pass over dqkv
            dqkv_cols = 3 * c.hd
            part = (self._csum_qkv[:c.tokens // 32 * dqkv_cols] if self.fold_defer
                    else self._colsum_part(c.tokens, dqkv_cols))
            dqkv = self._attn_bwd(do, att, delta=delta, colsum=part)
            self._mm_dw("qkv.dW", dqkv, h1, G["qkv_w"])
            if self.fold_defer:
                folds.append((part, c.tokens // 32, dqkv_cols, G["qkv_b"]))
            else:
                kernels.colsum_fold(part, c.tokens // 32, dqkv_cols, G["qkv_b"])
        else:
            do = self._mm_dx("proj.dx", dx2, P["proj_w"])
            dqkv = self._attn_bwd(do, att)
            self._mm_dw("qkv.dW", dqkv, h1, G["qkv_w"])
            kernels.bias_grad(dqkv, G["qkv_b"], ws)
        dh1 = self._mm_dx("qkv.dx", dqkv, P["qkv_w"])
        dx = torch.empty_like(dh1)
        # ... and LN1 backward sums dres = dx2: the proj bias gradient
        self._ln_bwd_fold(folds, 1, dh1, x, P["ln1_w"], m1, r1, dx, G["ln1_w"], G["ln1_b"],
                          dres=dx2, dres_sum=G["proj_b"])
        if folds:
            kernels.fold_sets(folds)
        return dx

    def _ln_bwd_fold(self, folds, k, dy, x, w, mean, rstd, dx, dgamma, dbeta, dres, dres_sum):
        """LayerNorm backward; with fold_defer its dgamma / dbeta / dres-sum folds join the
        block's fold list (partials in the k-th LN partial buffer) instead of launching."""
        if not self.fold_defer:
            kernels.ln_bwd(dy, x, w, mean, rstd, dx, dgamma, dbeta, self.ws, dres=dres,
                           dres_sum=dres_sum)
            return
        part = self._lnpart[k]
        P = kernels.ln_bwd_partials(dy, x, w, mean, rstd, dx, part, dres=dres, dres_sum=True)
        H = x.shape[-1]
        for i, out in enumerate((dgamma, dbeta, dres_sum)):
            folds.append((part[i * P * H:(i + 1) * P * H], P, H, out))

    def _block_bwd(self, dy, cache, P, G):
        if self.fused:
            return self._block_bwd_fused(dy, cache, P, G)
        hd = self.cfg.hd
        x, h1, m1, r1, att, o, x2, h2, m2, r2, u, a = cache
        torch.mm(dy.t(), a, out=G["fc2_w"])
        torch.sum(dy, 0, out=G["fc2_b"])
        da = torch.mm(dy, P["fc2_w"])
        du = torch.ops.aten.gelu_backward(da, u, approximate="tanh")
        torch.mm(du.t(), h2, out=G["fc1_w"])
        torch.sum(du, 0, out=G["fc1_b"])
        dh2 = torch.mm(du, P["fc1_w"])
        dx2, dw, db = torch.ops.aten.native_layer_norm_backward(
            dh2, x2, (hd,), m2, r2, P["ln2_w"], P["ln2_b"], [True, True, True])
        G["ln2_w"].copy_(dw)
        G["ln2_b"].copy_(db)
        dx2 += dy
        torch.mm(dx2.t(), o, out=G["proj_w"])
        torch.sum(dx2, 0, out=G["proj_b"])
        do = torch.mm(dx2, P["proj_w"])
        dqkv = self._attn_bwd(do, att)
        torch.mm(dqkv.t(), h1, out=G["qkv_w"])
        torch.sum(dqkv, 0, out=G["qkv_b"])
        dh1 = torch.mm(dqkv, P["qkv_w"])
        dx, dw, db = torch.ops.aten.native_layer_norm_backward(
            dh1, x, (hd,), m1, r1, P["ln1_w"], P["ln1_b"], [True, True, True])
        G["ln1_w"].copy_(dw)
        G["ln1_b"].copy_(db)
        dx += dx2
        return dx

    def _head_fwd_bwd(self, x, PF, PE, G, targets, wte_acc):
        """Final LN + tied LM head + mean token CE; returns (loss, dx). Fills
        G (final bucket grads) and wte_acc (fp32 head contribution to wte)."""
        if self.fused:
            return self._head_fused(x, PF, PE, G, targets, wte_acc)
        hd = self.cfg.hd
        hf, mf, rf = torch.native_layer_norm(x, (hd,), PF["lnf_w"], PF["lnf_b"], LN_EPS)
        logits = torch.mm(hf, PE["wte"].t()).float()
        tgt = targets.reshape(-1)
        T = tgt.numel()
        lse = torch.logsumexp(logits, -1)
        loss = (lse - logits.gather(1, tgt[:, None]).squeeze(1)).sum() / T
        p = torch.exp(logits - lse[:, None])
        p[torch.arange(T, device=p.device), tgt] -= 1.0
        dlog = (p / T).to(self.cdt)
        del logits, p
        if self.cdt == torch.float32:
            torch.mm(dlog.t(), hf, out=wte_acc)
        else:
            wte_acc.copy_(torch.ops.aten.mm.dtype(dlog.t(), hf, torch.float32))
        dhf = torch.mm(dlog, PE["wte"])
        dx, dw, db = torch.ops.aten.native_layer_norm_backward(
            dhf, x, (hd,), mf, rf, PF["lnf_w"], PF["lnf_b"], [True, True, True])
        G["lnf_w"].copy_(dw)
        G["lnf_b"].copy_(db)
        return loss, dx

    def _head_fused(self, x, PF, PE, G, targets, wte_acc):
        """libzinf LN + one-pass softmax cross-entropy over bf16 logits (in place:
        the logits buffer becomes dlogits); the tied-head GEMMs on their sites' choice."""
        _, hf, mf, rf = self._ln(x, PF["lnf_w"], PF["lnf_b"])
        logits = torch.empty(hf.shape[0], PE["wte"].shape[0], dtype=hf.dtype, device=hf.device)
        if self._zi("head.fwd", hf, PE["wte"], logits):
            kernels.gemm_sk(hf, PE["wte"], logits)
        else:
            torch.mm(hf, PE["wte"].t(), out=logits)
        tgt = targets.reshape(-1)
        T = tgt.numel()
        rows = torch.empty(T, dtype=torch.float32, device=x.device)
        loss = torch.empty((), dtype=torch.float32, device=x.device)
        kernels.softmax_ce(logits, tgt, rows, loss, 1.0 / T)
        dlog = logits
        self._mm_dw("head.dW", dlog, hf, wte_acc)
        dhf = self._mm_dx("head.dx", dlog, PE["wte"])
        del logits, dlog
        dx = torch.empty_like(dhf)
        kernels.ln_bwd(dhf, x, PF["lnf_w"], mf, rf, dx, G["lnf_w"], G["lnf_b"], self.ws)
        return loss, dx

    # ------------------------------------------------------------------- reduce
    def _grad_views(self, li, b: Bucket, slot: int) -> tuple[dict, torch.Tensor]:
        if self.cdt != self.half:
            flat = self.gwide[li] if b.key != "embed" else torch.zeros(
                b.shard * self.N, dtype=self.cdt, device=self.dev)
        else:
            flat = self.gembed[li] if b.key == "embed" else self.gslots[li][slot]
        return self._params(b, flat), flat

    def _contrib(self, li, b: Bucket, slot: int) -> torch.Tensor:
        return self.gembed[li] if b.key == "embed" else self.gslots[li][slot]

    def _finish_grad(self, li, b: Bucket, slot: int, flat: torch.Tensor):
        """Cast the compute-dtype grads to the half contribution (RNE)."""
        dst = self._contrib(li, b, slot)
        if flat.data_ptr() != dst.data_ptr():
            kernels.cast_f32_to_half(flat[:b.numel].contiguous(), dst[:b.numel])
        if b.shard * self.N > b.numel:
            dst[b.numel:b.shard * self.N].zero_()

    def _reduce_update(self, b: Bucket, slot: int, consts):
        """zi_rs_adam for every local rank's shard of bucket b.

        Runs on the optimizer stream, overlapped with the next bucket's backward
        GEMMs (PAPER §6.2: reduce-scatter of op i+1 || compute of op i): the
        fused RS + Adam is HBM-bound, the GEMMs tensor-bound. The gradient slot
        is handed back through ``gfree``; with peers (DistComm) it is free only
        once every rank finished reading it, i.e. after the next bucket's
        opt-stream barrier (channel 2), which follows each rank's RS of b.
        """
        cur = torch.cuda.current_stream()
        os_ = self.opt_stream if self.overlap_opt else cur
        if os_ is not cur:
            os_.wait_stream(cur)              # bucket b's gradients are complete
        key = "embed" if b.key == "embed" else slot
        if self.comm.is_local:
            contribs = [self._contrib(li, b, slot) for li in range(len(self.ranks))]
        else:
            self.comm.device_barrier(os_, channel=2)
            if self._pending_free is not None:   # peers are done with the previous slot
                ev = torch.cuda.Event()
                ev.record(os_)
                self.gfree[self._pending_free] = ev
            self._pending_free = key
            contribs = list(self.peer_gembed) if b.key == "embed" else list(self.peer_gslots[slot])
        scale = 1.0 / self.N
        if self.offload:
            self._reduce_update_offload(b, slot, consts, contribs, scale)
            return
        if self.nvme:  # the streamer thread runs nc -> cg -> RS+Adam -> D2H -> nc
            ready = torch.cuda.Event()
            ready.record(cur)
            self._nvme_wait[key] = [
                self.streamer.submit(b, li, r, contribs, scale, ready,
                                     self._shard_view(self.p16, li, b))
                for li, r in enumerate(self.ranks)]
            return
        host_params = self.host_params
        with torch.cuda.stream(os_):
            t0 = self._tmark(os_)
            for li, r in enumerate(self.ranks):
                p16 = self._shard_view(self.p16, li, b)
                ph = torch.empty(b.shard, dtype=self.half, device=self.dev) if host_params else p16
                kernels.rs_adam_dc(contribs, r * b.shard, b.shard, b.numel, scale,
                                   self._shard_view(self.p32, li, b),
                                   self._shard_view(self.m, li, b),
                                   self._shard_view(self.v, li, b), ph,
                                   self.adam, g_out=self._gout(li, b))
                if host_params:  # updated bf16 shard back to its pinned home (D2H)
                    p16.copy_(ph, non_blocking=True)
            self._tspan(b.op, "reduce_scatter", t0, self._tmark(os_))
            if self.comm.is_local and os_ is not cur:
                ev = torch.cuda.Event()
                ev.record(os_)
                self.gfree[key] = ev

    def _ostate_prefetch(self) -> None:
        """Issue the H2D of the backward's first NS-1 optimizer-state chunks (cg lane)."""
        ph = self._phase
        self._phase = "backward"
        for q in range(len(self.stage) - 1):
            self._ostate_h2d(q)
        self._phase = ph

    def _ostate_h2d(self, q: int, stream=None) -> None:
        """Issue the H2D of this step's optimizer-state chunk q into its staging slot
        (the cg lane, or ``stream``), behind the D2H that last drained the slot."""
        if q >= len(self._ochunks) or q in self._oh2d:
            return
        b, li, s, n = self._ochunks[q]
        k = (self._obase + q) % len(self.stage)
        h2d = stream if stream is not None else self.h2d_stream
        with torch.cuda.stream(h2d):
            if self.ev_d2h[k] is not None:
                h2d.wait_event(self.ev_d2h[k])     # staging slot drained
            t0 = self._tmark(h2d)
            for dst, a in zip(self.stage[k], (self.p32, self.m, self.v)):
                dst[:n].copy_(self._shard_view(a, li, b)[s:s + n], non_blocking=True)
            self._tspan(b.op, "cg", t0, self._tmark(h2d))
            ev = torch.cuda.Event()
            ev.record(h2d)
        self._oh2d[q] = ev

    def _reduce_update_offload(self, b: Bucket, slot: int, consts, contribs, scale: float):
        """Optimizer states in pinned host DRAM (PAPER §5.1.1).

        The bucket's chunks stream through the HBM staging ring:
        H2D(q+NS-1) on the h2d stream || zi_rs_adam(q) on the optimizer stream ||
        D2H(q-1) on the d2h stream — three engines busy at once, the compute
        stream never waits on PCIe. The first NS-1 chunks of a step are
        prefetched when the step starts (during the forward), and the last
        chunks' D2H drains during the next forward (``defer_writeback``), so
        the PCIe lanes stay busy across the step boundary. The bf16 param shard
        is updated in place in HBM (or staged back to host when params are
        offloaded too).
        """
        cur = torch.cuda.current_stream()
        opt, d2h = self.opt_stream, self.d2h_stream
        opt.wait_stream(cur)                 # grads of bucket b are complete
        host_params = self.host_params
        NS = len(self.stage)
        gouts = {li: self._gout(li, b) for li in range(len(self.ranks))}
        for q in self._obucket[b.key]:
            _, li, s, n = self._ochunks[q]
            r = self.ranks[li]
            L = b.shard
            hp, hm, hv = (self._shard_view(a, li, b) for a in (self.p32, self.m, self.v))
            p16 = self._shard_view(self.p16, li, b)
            k = (self._obase + q) % NS
            self._ostate_h2d(q)
            self._ostate_h2d(q + NS - 1)
            sp, sm, sv = (x[:n] for x in self.stage[k])
            with torch.cuda.stream(opt):
                opt.wait_event(self._oh2d.pop(q))
                ph = self.stage16[k][:n] if host_params else p16[s:s + n]
                go = gouts[li]
                kernels.rs_adam_dc(contribs, r * L + s, n, b.numel, scale, sp, sm, sv, ph,
                                   self.adam, g_out=go[s:s + n] if go is not None else None)
                ev_c = torch.cuda.Event()
                ev_c.record(opt)
            if host_params:   # bf16 write-back on its own lane: the next fetch waits on it only
                p16s = self.p16_stream
                with torch.cuda.stream(p16s):
                    p16s.wait_event(ev_c)
                    p16[s:s + n].copy_(self.stage16[k][:n], non_blocking=True)
                    ev_p = torch.cuda.Event()
                    ev_p.record(p16s)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_c)
                t0 = self._tmark(d2h)
                for dst, src in zip((hp, hm, hv), (sp, sm, sv)):
                    dst[s:s + n].copy_(src, non_blocking=True)
                self._tspan(b.op, "grad_offload", t0, self._tmark(d2h))
                if host_params:
                    d2h.wait_event(ev_p)      # slot k (stage16 too) is drained
                ev_d = torch.cuda.Event()
                ev_d.record(d2h)
            self.ev_d2h[k] = ev_d
            self.offload_bytes += 2 * 12 * n + (2 if host_params else 0) * n
        ev_free = torch.cuda.Event()
        ev_free.record(opt)
        self.gfree["embed" if b.key == "embed" else slot] = ev_free
        if host_params:
            ev = torch.cuda.Event()
            ev.record(self.p16_stream)
            if self.nvme_params:   # nc lane, write direction: the shard file is updated from
                self.p16_ready.pop(b.key, None)   # the arena once the D2H landed; the next
                for li, r in enumerate(self.ranks):   # step's nc read of b waits on it
                    self._p16_wfut[(b.key, r)] = self._io.submit(
                        self._wb_job, self._pkey(b, r), self._shard_view(self.p16, li, b), ev)
            else:
                self.p16_ready[b.key] = ev

    @property
    def defer_writeback(self) -> bool:
        """Optimizer-offload steps end when the last rs_adam is done, not when its
        D2H landed: the fp32 write-back drains during the next forward, which reads
        only the bf16 params — updated in HBM, or, with params on the host, written
        back on their own lane and awaited per bucket by the next fetch (p16_ready).
        Not with host checkpoints (d2h stream shared) or under graph capture (every
        side stream must rejoin)."""
        return (self.offload and self.act_ckpt != "host"
                and not torch.cuda.is_current_stream_capturing())

    def flush(self) -> None:
        """Order the current stream after every in-flight host transfer (the deferred
        optimizer-state write-back); host-side readers then synchronize as usual."""
        cur = torch.cuda.current_stream()
        cur.wait_stream(self.d2h_stream)
        cur.wait_stream(self.h2d_stream)
        cur.wait_stream(self.p16_stream)
        if self.nvme_params:   # the bf16 param files hold the last update
            for f in list(self._p16_wfut.values()):
                f.result()

    # ------------------------------------------------- activation checkpoints (PAPER §5.1.2)
    def _ckpt_save(self, li: int, i: int, x_in: torch.Tensor):
        """Keep block i's input as its checkpoint: in HBM, or D2H to pinned host."""
        if self.act_ckpt == "device":
            return x_in
        d2h, cur = self.d2h_stream, torch.cuda.current_stream()
        d2h.wait_stream(cur)                      # x_in is produced on the compute stream
        with torch.cuda.stream(d2h):
            t0 = self._tmark(d2h)
            self.ckpt_host[li][i].copy_(x_in.view(-1), non_blocking=True)
            self._tspan(self.buckets[1 + i].op, "grad_offload", t0, self._tmark(d2h))
            ev = torch.cuda.Event()
            ev.record(d2h)
        x_in.record_stream(d2h)                   # no reuse of its memory before the copy
        self._ckpt_saved[(li, i)] = ev
        self.ckpt_bytes += x_in.numel() * x_in.element_size()
        return None

    def _ckpt_prefetch(self, li: int, i: int) -> None:
        """H2D of block i's checkpoint into its ring slot, one block ahead of use."""
        h2d, cur = self.h2d_stream, torch.cuda.current_stream()
        dst = self.ckpt_ring[li][i % 2]
        h2d.wait_stream(cur)                      # the slot's previous block is recomputed
        with torch.cuda.stream(h2d):
            h2d.wait_event(self._ckpt_saved.pop((li, i)))
            t0 = self._tmark(h2d)
            dst.view(-1).copy_(self.ckpt_host[li][i], non_blocking=True)
            self._tspan(self.buckets[1 + i].op, "cg", t0, self._tmark(h2d))
            ev = torch.cuda.Event()
            ev.record(h2d)
        self._ckpt_loaded[(li, i)] = ev
        self.ckpt_bytes += dst.numel() * dst.element_size()

    def _ckpt_get(self, li: int, i: int, cached):
        if self.act_ckpt == "device":
            return cached
        if (li, i) not in self._ckpt_loaded:      # the last block: not prefetched yet
            self._ckpt_prefetch(li, i)
        torch.cuda.current_stream().wait_event(self._ckpt_loaded.pop((li, i)))
        return self.ckpt_ring[li][i % 2]

    def _wait_gslot(self, slot) -> None:
        """Before overwriting a gradient slot: the optimizer stream must be done reading it."""
        for done in self._nvme_wait.pop(slot, ()):   # NVMe streamer jobs still using it
            done.wait()
            if self.streamer.err is not None:         # surface the I/O failure itself
                raise self.streamer.err
            torch.cuda.current_stream().wait_event(done.ev)
        ev = self.gfree.pop(slot, None)
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def _gout(self, li, b):
        if getattr(self, "capture_grads", False):
            g = torch.empty(b.shard, dtype=torch.float32, device=self.dev)
            self.grad_shards.setdefault(b.key, {})[self.ranks[li]] = g
            return g
        return None

    # --------------------------------------------------------------------- step
    def step(self, batches) -> torch.Tensor:
        """One partitioned training step; ``batches[li] = (tokens, targets)``
        (int64 [batch, seq] CUDA tensors) for each local rank. Returns the
        mean loss over all ranks as a 0-d fp32 CUDA tensor. ``self.launches`` counts the
        libzinf kernels the step launched (the library's own counter, zi_launch_count)."""
        n0 = _lib.launch_count()
        loss = self._step(batches)
        self.launches += _lib.launch_count() - n0
        return loss

    def _step(self, batches) -> torch.Tensor:
        c = self.cfg
        self.t += 1
        consts = None                 # Adam constants live on the device (self.adam)
        self.grad_shards = {}
        cur = torch.cuda.current_stream()
        self.adam.advance()           # t += 1 and this step's bias corrections, on the GPU
        gs = self.gather_stream if self.prefetch else cur
        nloc = len(self.ranks)
        if not self.comm.is_local and self.N > 1:
            self.comm.device_barrier()  # peers' previous-step Adam writes are done
        if self.offload:
            # the cg lane follows this step's start (under capture: joins the graph)
            self.h2d_stream.wait_stream(cur)
            if not self.defer_writeback and not torch.cuda.is_current_stream_capturing():
                # last step's host writes landed (a graph replay follows the previous
                # replay, which joined every lane, in stream order)
                self.h2d_stream.wait_stream(self.d2h_stream)
            self._obase += len(self._ochunks)
            self._oh2d = {}
        self._spans = []
        self._pending_free = None
        # events of the previous step are complete (cur joined every side stream at its
        # end) and must not leak into a graph capture
        self.gfree.clear()
        self.events.clear()
        if torch.cuda.is_current_stream_capturing():
            # host-side synchronized before capture: drop events recorded outside it
            self.p16_ready.clear()
            if self.offload:
                self.ev_d2h = [None] * len(self.ev_d2h)
        self._ckpt_saved.clear()
        self._ckpt_loaded.clear()
        # the step's fetch positions and their nc / cg / gg plan
        if self._fplan is None:
            from .schedule import Op, OperatorSequence
            ops = tuple(Op(b.op, (b.key,), 2 * b.numel, 1) for b in self._flist)
            self._fplan = plan_prefetch(OperatorSequence(ops, "step"), self.depths)
        self._fpos = 0
        self.issue_log = []
        self._staged.clear()
        self._cg_ev.clear()
        self._cg_issued.clear()
        self._nc_fut.clear()
        self._nc_issued.clear()
        if torch.cuda.is_current_stream_capturing():
            self._cg_free.clear()      # recorded outside the capture (and complete)
        if self.host_params:
            self.h2d_stream.wait_stream(cur)   # the cg lane forks from this step's start
        self._nvme_wait = {}
        self._t0 = self._tmark(cur)
        host_params = self.host_params
        if self.offload and not host_params:   # state prefetch for the backward, during the forward
            self._ostate_prefetch()
        self._phase = "forward"
        gs.wait_stream(cur)
        blocks = self.buckets[1:-1]
        E, FB = self.buckets[0], self.buckets[-1]
        # ---- forward
        self._fetch(E, 0, gs)
        if blocks:
            self._fetch(blocks[0], 0, gs)
        PE = self._params(E, self._full(E, 0))
        c0 = self._tmark(cur)
        xs = [self._embed_fwd(PE, batches[li][0]) for li in range(nloc)]
        self._tspan(E.op, "compute", c0, self._tmark(cur))
        caches = [[None] * len(blocks) for _ in range(nloc)]
        ev_every, fq = self.fwd_state_prefetch_every, 0
        nb = len(blocks)
        for i, b in enumerate(blocks):
            full = self._full(b, self._pslot(i, nb))
            if i + 1 < len(blocks):
                gs.wait_stream(cur)  # ring slot (i+1)%2 was last read by compute of block i-1
                self._fetch(blocks[i + 1], self._pslot(i + 1, nb), gs)
                if (self.offload and host_params and ev_every and i % ev_every == ev_every - 1
                        and fq < len(self.stage) - 1):   # slots this step has not claimed
                    # the H2D lane has slack while the forward computes: queue one
                    # optimizer-state chunk behind this fetch, in the fetch's own FIFO
                    # (so it never delays the next fetch by more than its own length)
                    self._phase = "backward"
                    self._ostate_h2d(fq, stream=gs)
                    self._phase = "forward"
                    fq += 1
            else:
                gs.wait_stream(cur)
                self._phase = "backward"     # the head is the first backward op
                self._fetch(FB, self._pslot(nb, nb), gs)
                if self.offload and host_params:
                    # with params on the host the forward's H2D lane carries their fetches;
                    # the state prefetch starts behind the last of them
                    self._ostate_prefetch()
                self._phase = "forward"
            P = self._params(b, full)
            c0 = self._tmark(cur)
            for li in range(nloc):
                x_in = xs[li]
                xs[li], caches[li][i] = self._block_fwd(x_in, P)
                if self.act_ckpt is not None:   # keep only the block input (checkpoint)
                    caches[li][i] = self._ckpt_save(li, i, x_in)
            self._tspan(b.op, "compute", c0, self._tmark(cur))
        fslot = len(blocks) % 2                 # the head's gradient slot
        self._phase = "backward"
        if not blocks:
            self._fetch(FB, 0, gs)
        PF = self._params(FB, self._full(FB, self._pslot(nb, nb) if blocks else 0))
        # ---- head (forward + backward fused; its bucket reduces first)
        losses = []
        GF = []
        self._wait_gslot(fslot)
        c0 = self._tmark(cur)
        for li in range(nloc):
            G, flat = self._grad_views(li, FB, fslot)
            loss, xs[li] = self._head_fwd_bwd(xs[li], PF, PE, G, batches[li][1], self.wte_acc[li])
            self._finish_grad(li, FB, fslot, flat)
            losses.append(loss)
        self._tspan(FB.op, "compute", c0, self._tmark(cur))
        self._reduce_update(FB, fslot, consts)
        # ---- backward through the blocks, re-gathering each one
        # blocks[-1] is still in its slot from the forward (the head used another), and
        # so are the reuse-cached blocks: the backward fetches only blocks[: nb - 1 - K]
        for j in range(nb - 1, -1, -1):
            b = blocks[j]
            slot = j % 2                           # gradient slot
            full = self._full(b, self._pslot(j, nb))
            if j - 1 >= 0 and j - 1 < nb - 1 - self.K:
                gs.wait_stream(cur)
                self._fetch(blocks[j - 1], self._pslot(j - 1, nb), gs)
            P = self._params(b, full)
            self._wait_gslot(slot)
            if self.act_ckpt == "host" and j - 1 >= 0:
                for li in range(nloc):          # prefetch the next checkpoint (cg lane)
                    self._ckpt_prefetch(li, j - 1)
            c0 = self._tmark(cur)
            for li in range(nloc):
                G, flat = self._grad_views(li, b, slot)
                cache = caches[li][j]
                if self.act_ckpt is not None:   # recompute the block from its checkpoint
                    _, cache = self._block_fwd(self._ckpt_get(li, j, cache), P)
                xs[li] = self._block_bwd(xs[li], cache, P, G)
                caches[li][j] = cache = None
                self._finish_grad(li, b, slot, flat)
            self._tspan(b.op, "compute", c0, self._tmark(cur))
            self._reduce_update(b, slot, consts)
        # ---- embedding backward: tied wte = head part + scatter of dx
        self._wait_gslot("embed")
        c0 = self._tmark(cur)
        for li in range(nloc):
            G, flat = self._grad_views(li, E, 0)
            tok = batches[li][0].reshape(-1)
            # tied wte: head contribution + the lookup's gradient rows, summed per vocabulary
            # row in sequence order (zi_embed_grad: no float atomics) and rounded to half
            if G["wte"].dtype == torch.float32:
                wte16 = torch.empty(c.vocab, c.hd, dtype=self.half, device=self.dev)
                kernels.embed_grad(tok, xs[li].contiguous(), self.wte_acc[li], wte16, self.emb_work)
                kernels.cast_half_to_f32(wte16.view(-1), G["wte"].view(-1))
            else:  # fp32 accumulators -> RNE half contributions
                kernels.embed_grad(tok, xs[li].contiguous(), self.wte_acc[li], G["wte"],
                                   self.emb_work)
            # wpe: fixed-order fp32 batch sum, stored in the gradient's dtype (one pass)
            kernels.pos_grad(xs[li].contiguous().view(-1, c.hd), c.batch, G["wpe"])
            self._finish_grad(li, E, 0, flat)
        self._tspan(E.op, "compute", c0, self._tmark(cur))
        self._reduce_update(E, 0, consts)
        if self.nvme:
            self.streamer.drain()         # every bucket's states are back on NVMe
        if self.overlap_opt or self.offload:   # (an unused side stream must not be joined
            cur.wait_stream(self.opt_stream)  # under capture) the step ends when the last
                                              # bucket is updated
        if (self.offload and not self.defer_writeback) or self.nvme or self.act_ckpt == "host":
            cur.wait_stream(self.d2h_stream)  # ... and host transfers landed
            cur.wait_stream(self.h2d_stream)
            if self.offload and self.host_params:
                cur.wait_stream(self.p16_stream)
                self.p16_ready.clear()
        if gs is not cur:
            cur.wait_stream(gs)       # join the gather stream (required for graph capture)
        total = losses[0].float()
        for l in losses[1:]:
            total = total + l.float()
        return total / nloc if self.comm.is_local else total

    def step_graphed(self, batches) -> torch.Tensor:
        """``step`` captured once into a CUDA graph and replayed.

        The step's ~1000 launches (GEMMs, attention, libzinf kernels, the
        gathers and offload copies on their side streams) become one graph
        launch; Adam's per-step constants come from the device counter
        (zi_adam_advance inside the graph), tokens from static buffers the
        caller's batch is copied into. The first call warms up with two eager
        steps (real training steps) and captures; every call then replays.
        """
        cur = torch.cuda.current_stream()
        if self.nvme or self.nvme_params:   # host-thread NVMe I/O cannot live in a graph
            return self.step(batches)
        if self._graph is None:
            if self.trace:
                raise ValueError("tracing is not supported under graph capture")
            self._static = [(t.clone(), y.clone()) for t, y in batches]
            # warm cuBLAS / cuDNN plans and the allocator with two eager steps on a
            # snapshot of the model state, then restore it: every call of
            # step_graphed is exactly one training step
            self.flush()                 # no deferred write-back in flight under the snapshot
            torch.cuda.synchronize()
            state = [self.p16, self.p32, self.m, self.v, self.adam.step, self.adam.consts]
            snap = [s.clone() for s in state]
            for _ in range(2):
                self.step(self._static)
            torch.cuda.synchronize()
            multi = not self.comm.is_local and self.N > 1
            if multi:   # peers finished reading our buffers before we restore them ...
                self.comm.host_barrier()
            for s, c in zip(state, snap):
                s.copy_(c)
            del snap
            self.t -= 2
            torch.cuda.synchronize()
            if multi:   # ... and every rank restored before anyone replays (P2P reads)
                self.comm.host_barrier()
            g = torch.cuda.CUDAGraph()
            l0, t0 = self.launches, self.t
            if multi:
                self.comm.begin_capture()
            with torch.cuda.graph(g):
                self._static_loss = self.step(self._static)
                if multi:   # every side stream joined cur: pad the barrier parity there
                    self.comm.end_capture()
            self._graph = g
            self._launches_per_replay = self.launches - l0
            self.launches, self.t = l0, t0      # capture executes nothing
        for (st, sy), (t, y) in zip(self._static, batches):
            st.copy_(t, non_blocking=True)
            sy.copy_(y, non_blocking=True)
        self._graph.replay()
        self.t += 1
        self.launches += self._launches_per_replay
        return self._static_loss

    # ------------------------------------------------------------------ access
    def gathered(self, key: str) -> torch.Tensor:
        """Full half bucket (all ranks local) — for tests."""
        b = self.by_key[key]
        if self.offload:
            self.flush()        # host params: the deferred bf16 write-back has landed
        out = torch.empty(b.shard * self.N, dtype=self.half, device=self.dev)
        shards = [self._shard_view(self.p16, li, b).to(self.dev) for li in range(len(self.ranks))]
        kernels.allgather(shards, b.shard, out, b.numel)
        return out[:b.numel]

    def shard(self, key: str, li: int = 0) -> dict:
        b = self.by_key[key]
        if self.nvme:   # fp32 states read back from their .shard files
            from .store import TierKind as TK
            r = self.ranks[li]
            out = {n: self.store.read(self.streamer.key(key, n, r), TK.NVME).wait()
                   for n in ("p32", "m", "v")}
            out["p16"] = self._shard_view(self.p16, li, b)
            return out
        if self.offload:
            self.flush()
            torch.cuda.current_stream().synchronize()   # host states: write-back landed
        return {n: self._shard_view(a, li, b) for n, a in
                (("p16", self.p16), ("p32", self.p32), ("m", self.m), ("v", self.v))}

    def param_file_shard(self, key: str, li: int = 0) -> torch.Tensor:
        """Params on NVMe: rank li's bf16 shard of bucket ``key`` as its .shard file holds it."""
        self.flush()
        return self.pstore.read(self._pkey(self.by_key[key], self.ranks[li]), TierKind.NVME).wait()

    def close(self) -> None:
        """Stop the NVMe streamer thread (it references the engine) and its store."""
        if self.nvme and self.streamer is not None:
            self.streamer.close()
            self.store.close()
            self.streamer = None
        if self.nvme_params and self._io is not None:
            self.flush()
            self._io.shutdown(wait=True)
            self.pstore.close()
            self._io = None


def synthetic_tokens(cfg: GPTConfig, seed: int, rank: int, step: int = 0, device="cuda"):
    """Uniform token ids on [0, V) per (rank, step) — same generator as the oracle."""
    import numpy as np
    rng = np.random.default_rng([seed, rank, step])
    tok = rng.integers(0, cfg.vocab, size=(cfg.batch, cfg.seq + 1), dtype=np.int64)
    t = torch.from_numpy(tok)
    return t[:, :-1].contiguous().to(device), t[:, 1:].contiguous().to(device)
