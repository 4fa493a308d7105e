"""Placement planner: feasibility, maximum model size, effective bandwidth and strategy
ranking across the paper's device-placement strategies, with a DGX-2 profile (the SPEC's
default) and a measured B200 profile (SPEC.md placement-planner
module, the text around SPEC.md:263-311; PAPER Table 3, Fig. 9, §6.1, Table 4).

Host-side analytics only: nothing here runs in the training step. The engine's own
placement knobs (``gpt.Placement``, ``param_cache``) are the executed counterpart; the
planner says which of them a model needs on a cluster and what efficiency the paper's
bandwidth model predicts for it.

The memory terms restate the reference's memory model (``memory.py:83-121``: 12·nl·hd²
parameters, 20 B/param of model states, MSWM = 16·hd², AWM = 2·ci·bsz·seq·(16·hd +
2·heads·seq) bytes) and the efficiency terms its bandwidth model (``efficiency.py``:
ait = seq·bsz, seq·bsz/4, 24·hd·ci; efficiency = ait·bw / (ait·bw + peak)).
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

GB = 1e9

# bytes per parameter of the model states (memory.py:17-25): fp16 p, g; fp32 m, v, master, grad
STATE_BYTES = 20
FRAMEWORK_RESERVE = 2e9      # SPEC DESIGN DECISIONS: fixed per-device working reserve


@dataclass(frozen=True)
class ClusterConfig:
    """SPEC ClusterConfig; bandwidths in bytes/s (decimal), capacities in bytes."""
    nodes: int = 1
    devices_per_node: int = 16
    device_mem_bytes: float = 32e9
    host_mem_bytes_per_node: float = 1.5e12
    nvme_bytes_per_node: float = 28e12
    pcie_bw_per_device: float = 12e9
    host_mem_bw_per_node: float = 48e9        # the node's shared PCIe path to host memory
    nvme_bw_per_node: float = 25e9
    device_device_bw: float = 300e9
    peak_tp_per_device: float = 70e12
    name: str = "dgx2"

    def __post_init__(self):
        for k in ("nodes", "devices_per_node", "device_mem_bytes", "host_mem_bytes_per_node",
                  "nvme_bytes_per_node", "pcie_bw_per_device", "host_mem_bw_per_node",
                  "nvme_bw_per_node", "device_device_bw", "peak_tp_per_device"):
            if not getattr(self, k) > 0:
                raise ValueError(f"ClusterConfig.{k} must be positive")

    @property
    def world_size(self) -> int:
        return self.nodes * self.devices_per_node

    @classmethod
    def from_flat(cls, kv: dict) -> "ClusterConfig":
        """The flat profile keys of the SPEC's external interface."""
        m = {"nodes": "nodes", "devices_per_node": "devices_per_node",
             "device_mem": "device_mem_bytes", "host_mem_per_node": "host_mem_bytes_per_node",
             "nvme_per_node": "nvme_bytes_per_node", "pcie_bw": "pcie_bw_per_device",
             "host_bw_per_node": "host_mem_bw_per_node", "nvme_bw_per_node": "nvme_bw_per_node",
             "d2d_bw": "device_device_bw", "peak_tp": "peak_tp_per_device"}
        args = {}
        for k, v in kv.items():
            if k not in m:
                raise ValueError(f"unknown cluster key {k!r}")
            args[m[k]] = int(v) if m[k] in ("nodes", "devices_per_node") else float(v)
        return cls(**args)


def dgx2(nodes: int = 1) -> ClusterConfig:
    """The SPEC's default profile (16 V100-32GB per node; §6.1's 12 / 48 / 25 GB/s)."""
    return ClusterConfig(nodes=nodes)


def b200(nodes: int = 1, hbm_bytes: float = 180e9, host_link_gbs: float = 55.6,
         peak_tflops: float = 1386.0) -> ClusterConfig:
    """One 8 x B200 node per `nodes`. Measured on this pool's boxes: the pinned host link
    (bench `offload.host_link_peak`: 55.6 GB/s H2D per GPU) and the sustained dense bf16
    peak (MEASURED_PEAKS.json, 1386 TFLOPS). From the part: 180 GB HBM3e, NVLink 5 at
    900 GB/s per direction. Not measured here (one GPU per box): the node's aggregate
    host-memory path, taken as 8 independent links (bandwidth-centric partitioning, PAPER
    §6.1), 2 TB of host DRAM and 30 TB / 50 GB/s of local NVMe per node."""
    return ClusterConfig(nodes=nodes, devices_per_node=8, device_mem_bytes=hbm_bytes,
                         host_mem_bytes_per_node=2e12, nvme_bytes_per_node=30e12,
                         pcie_bw_per_device=host_link_gbs * GB,
                         host_mem_bw_per_node=8 * host_link_gbs * GB, nvme_bw_per_node=50e9,
                         device_device_bw=900e9, peak_tp_per_device=peak_tflops * 1e12,
                         name="b200")


class Tier(enum.Enum):
    DEVICE = "device"
    HOST = "host"
    NVME = "nvme"


class Strategy(enum.Enum):
    """PAPER Table 3 rows, in the SPEC's order (also the max-size monotonicity order)."""
    DATA_PARALLEL = "DataParallel"
    ZERO2 = "Zero2"
    ZERO_OFFLOAD = "ZeroOffload"
    THREE_D = "ThreeD"
    ZERO3 = "Zero3"
    ZERO_INF_CPU = "ZeroInfCpu"
    ZERO_INF_NVME = "ZeroInfNvme"


# (optimizer + gradient tier, partitioned?) x (parameter tier, partitioned?) — Table 3
PLACEMENT = {
    Strategy.DATA_PARALLEL: ((Tier.DEVICE, False), (Tier.DEVICE, False)),
    Strategy.ZERO2: ((Tier.DEVICE, True), (Tier.DEVICE, False)),
    Strategy.ZERO_OFFLOAD: ((Tier.HOST, True), (Tier.DEVICE, False)),
    Strategy.THREE_D: ((Tier.DEVICE, True), (Tier.DEVICE, True)),
    Strategy.ZERO3: ((Tier.DEVICE, True), (Tier.DEVICE, True)),
    Strategy.ZERO_INF_CPU: ((Tier.HOST, True), (Tier.HOST, True)),
    Strategy.ZERO_INF_NVME: ((Tier.NVME, True), (Tier.NVME, True)),
}


@dataclass(frozen=True)
class ModelShape:
    """memory.py's ModelConfig: nl blocks of hidden hd; bsz per device; ci blocks per
    activation checkpoint."""
    nl: int
    hd: int
    attn_heads: int = 32
    seq: int = 1024
    bsz: float = 1.0
    ci: int = 1

    @property
    def params(self) -> int:
        return 12 * self.nl * self.hd * self.hd


def mswm_bytes(hd: float, tiling: int = 1) -> float:
    """Model-state working memory: fp16 param + grad of the largest (hd -> 4hd) linear,
    16·hd² bytes (memory.py:109-111); memory-centric tiling divides it by the tile count."""
    return 16.0 * hd * hd / tiling


def awm_bytes(s: ModelShape, hd: float | None = None) -> float:
    """Activation working memory between two checkpoints (memory.py:99-121)."""
    h = s.hd if hd is None else hd
    return 2.0 * s.ci * s.bsz * s.seq * (16 * h + 2 * s.attn_heads * s.seq)


def working_memory(s: ModelShape, hd: float | None = None, tiling: int = 1) -> float:
    h = s.hd if hd is None else hd
    return mswm_bytes(h, tiling) + awm_bytes(s, h) + FRAMEWORK_RESERVE


# ---------------------------------------------------------------- bandwidth model
class AitKind(enum.Enum):
    PARAM_GRAD = "param_grad"
    OPTIMIZER_STATES = "optimizer_states"
    ACTIVATION_CKPT = "activation_ckpt"


def ait(kind: AitKind, s: ModelShape) -> float:
    """efficiency.py ait(): flops per byte moved for one iteration (8·bsz·seq·Ψ flops)."""
    if kind is AitKind.PARAM_GRAD:
        return float(s.seq * s.bsz)
    if kind is AitKind.OPTIMIZER_STATES:
        return float(s.seq * s.bsz) / 4.0
    return float(24 * s.hd * s.ci)


def efficiency(ait_value: float, bw: float, peak_tp: float) -> float:
    if not ait_value > 0 or not peak_tp > 0 or bw < 0:
        raise ValueError("efficiency: ait and peak must be positive, bw nonnegative")
    if math.isinf(bw):
        return 1.0
    return ait_value * bw / (ait_value * bw + peak_tp)


def required_bandwidth(ait_value: float, peak_tp: float, target_eff: float) -> float:
    if not 0 < target_eff < 1:
        raise ValueError("target efficiency must be in (0, 1)")
    return target_eff / (1 - target_eff) * peak_tp / ait_value


def effective_param_bandwidth(c: ClusterConfig, source: Tier, partitioned: bool) -> float:
    """Aggregate bandwidth at which a parameter reaches the devices (SPEC placement-planner,
    PAPER §6.1). Broadcast: one owner's path, constant in world size. Allgather: every
    device pulls its shard over its own link, bounded by each node's source bandwidth."""
    if source is Tier.DEVICE:
        src_node = c.device_device_bw * c.devices_per_node
    elif source is Tier.HOST:
        src_node = c.host_mem_bw_per_node
    else:
        src_node = c.nvme_bw_per_node
    if not partitioned:
        per_owner = src_node if source is not Tier.DEVICE else c.device_device_bw
        link = c.pcie_bw_per_device if source is not Tier.DEVICE else c.device_device_bw
        return min(link, per_owner)
    link = c.pcie_bw_per_device if source is not Tier.DEVICE else c.device_device_bw
    return min(c.world_size * link, c.nodes * src_node)


# ---------------------------------------------------------------- capacity model
def demands(psi: float, c: ClusterConfig, st: Strategy, wm: float,
            nvme_params: bool = True) -> dict:
    """Per-tier demand in bytes: device per device, host and NVMe per node (SPEC
    max_model_params post-condition and DESIGN DECISIONS)."""
    N, nodes = c.world_size, c.nodes
    dev, host, nvme = wm, 0.0, 0.0
    if st is Strategy.DATA_PARALLEL:
        dev += STATE_BYTES * psi
    elif st is Strategy.ZERO2:
        dev += 2 * psi + 18 * psi / N
    elif st is Strategy.ZERO_OFFLOAD:
        dev += 2 * psi
        host += 18 * psi / nodes
    elif st in (Strategy.THREE_D, Strategy.ZERO3):
        dev += STATE_BYTES * psi / N
    elif st is Strategy.ZERO_INF_CPU:
        host += STATE_BYTES * psi / nodes
    else:   # ZeroInfNvme: fp16 params on NVMe (Table 1 "NVMe NVMe") or staged in host
        if nvme_params:
            nvme += STATE_BYTES * psi / nodes
        else:
            nvme += 18 * psi / nodes
            host += 2 * psi / nodes
    return {Tier.DEVICE: math.ceil(dev), Tier.HOST: math.ceil(host), Tier.NVME: math.ceil(nvme)}


def capacities(c: ClusterConfig) -> dict:
    return {Tier.DEVICE: c.device_mem_bytes, Tier.HOST: c.host_mem_bytes_per_node,
            Tier.NVME: c.nvme_bytes_per_node}


def _fits(psi: float, c: ClusterConfig, st: Strategy, template: ModelShape, tiling: int,
          nvme_params: bool) -> bool:
    hd = math.sqrt(psi / (12.0 * template.nl))
    d = demands(psi, c, st, working_memory(template, hd, tiling), nvme_params)
    cap = capacities(c)
    return all(d[t] <= cap[t] for t in Tier)


def max_model_params(c: ClusterConfig, st: Strategy,
                     template: ModelShape = ModelShape(nl=128, hd=1), tiling: int = 1,
                     nvme_params: bool = True) -> int:
    """Largest Ψ that fits (monotone bisection over Ψ, 64 iterations, floored); hd follows
    Ψ at the template's depth. 0 if even Ψ = 1 does not fit."""
    if not _fits(1.0, c, st, template, tiling, nvme_params):
        return 0
    lo, hi = 1.0, 1.0
    while _fits(hi, c, st, template, tiling, nvme_params) and hi < 1e18:
        lo, hi = hi, hi * 2
    for _ in range(64):
        mid = (lo + hi) / 2
        if _fits(mid, c, st, template, tiling, nvme_params):
            lo = mid
        else:
            hi = mid
    return int(lo)


@dataclass
class FeasibilityReport:
    strategy: Strategy
    fits: bool
    demand: dict
    capacity: dict
    binding_constraint: str
    working_memory_ok: bool
    predicted_efficiency: float
    efficiency_by_kind: dict = field(default_factory=dict)


def _state_bw(c: ClusterConfig, tier: Tier) -> float:
    """Per-device bandwidth to where a state lives (device tier: not a transfer)."""
    if tier is Tier.DEVICE:
        return math.inf
    return effective_param_bandwidth(c, tier, True) / c.world_size


def feasibility(s: ModelShape, c: ClusterConfig, st: Strategy, tiling: int = 1,
                nvme_params: bool = True) -> FeasibilityReport:
    """Per-tier demand vs capacity for model `s` under strategy `st`; the predicted
    efficiency is the minimum over the three AIT kinds of the paper's bandwidth model at
    the bandwidth the strategy's placement gives each kind (per device)."""
    psi = s.params
    wm = working_memory(s, tiling=tiling)
    d = demands(psi, c, st, wm, nvme_params)
    cap = capacities(c)
    wm_ok = mswm_bytes(s.hd, tiling) + awm_bytes(s) + FRAMEWORK_RESERVE <= c.device_mem_bytes
    ratios = {t.value: d[t] / cap[t] for t in Tier}
    binding = max(ratios, key=ratios.get)
    fits = all(d[t] <= cap[t] for t in Tier) and wm_ok
    (opt_tier, _), (par_tier, par_part) = PLACEMENT[st]
    if par_tier is Tier.DEVICE and par_part:       # ZeRO-3 in HBM: allgather over NVLink
        pg_bw = effective_param_bandwidth(c, Tier.DEVICE, True) / c.world_size
    elif par_tier is Tier.DEVICE:
        pg_bw = math.inf
    else:
        pg_bw = effective_param_bandwidth(c, par_tier, True) / c.world_size
    act_bw = math.inf if st not in (Strategy.ZERO_INF_CPU, Strategy.ZERO_INF_NVME) \
        else c.pcie_bw_per_device       # checkpoints offloaded to host (PAPER §5.1.2)
    peak = c.peak_tp_per_device
    eff = {AitKind.PARAM_GRAD.value: efficiency(ait(AitKind.PARAM_GRAD, s), pg_bw, peak),
           AitKind.OPTIMIZER_STATES.value: efficiency(ait(AitKind.OPTIMIZER_STATES, s),
                                                      _state_bw(c, opt_tier), peak),
           AitKind.ACTIVATION_CKPT.value: efficiency(ait(AitKind.ACTIVATION_CKPT, s), act_bw, peak)}
    return FeasibilityReport(st, fits, {t.value: d[t] for t in Tier},
                             {t.value: cap[t] for t in Tier}, binding, wm_ok,
                             min(eff.values()), eff)


_TIER_PREF = {Strategy.DATA_PARALLEL: 0, Strategy.ZERO2: 0, Strategy.THREE_D: 0,
              Strategy.ZERO3: 0, Strategy.ZERO_OFFLOAD: 1, Strategy.ZERO_INF_CPU: 1,
              Strategy.ZERO_INF_NVME: 2}


def recommend(s: ModelShape, c: ClusterConfig, tiling: int = 1) -> list[FeasibilityReport]:
    """Strategies ranked by (fits, predicted efficiency, tier speed device > host > nvme),
    ties broken by the enum order (deterministic)."""
    order = list(Strategy)
    reps = [feasibility(s, c, st, tiling) for st in order]
    return sorted(reps, key=lambda r: (not r.fits, -r.predicted_efficiency,
                                       _TIER_PREF[r.strategy], order.index(r.strategy)))


def future_hardware_table(c: ClusterConfig, multipliers=(1, 10, 100), opt_ait: float = 512.0,
                          pg_ait: float = 1024.0, slow_eff: float = 0.9,
                          d2d_eff: float = 0.5) -> list[dict]:
    """PAPER Table 4: bandwidth needed when the device peak grows k-fold. Slow memory:
    aggregate = required_bandwidth(optimizer-state AIT, k·peak, slow_eff), per device =
    aggregate / world size; device-device = required_bandwidth(param+grad AIT, k·peak,
    d2d_eff). The default AITs are the SPEC's worked examples (512 = seq 1024 x bsz 2 / 4
    for the optimizer states, 1024 = seq 1024 x bsz 1 for parameters and gradients)."""
    rows = []
    for k in multipliers:
        peak = k * c.peak_tp_per_device
        agg = required_bandwidth(opt_ait, peak, slow_eff)
        rows.append({"multiplier": k, "slow_memory_per_device": agg / c.world_size,
                     "slow_memory_aggregate": agg,
                     "device_device": required_bandwidth(pg_ait, peak, d2d_eff)})
    return rows
