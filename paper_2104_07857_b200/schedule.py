"""Overlap-centric schedule: operator trace, prefetch plan, measured Timeline.

``trace_schedule`` records the operator sequence (PAPER §6.2 "constructing
an internal map of the operator sequence"); ``plan_prefetch`` decides, for
every op i, which later ops' fetch stages to issue while i runs — nc for
i+d_nc, cg for i+d_cg, gg for i+d_gg, default depths (3, 2, 1)
(SPEC.md:560-568). The engine executes the plan on side CUDA streams:

    nc  NVMe -> pinned host        (store worker threads)
    cg  pinned host -> HBM         (H2D copy-engine stream)
    gg  HBM shards -> full params  (gather stream: NVLink all-gather / P2P)

``Timeline`` holds either real intervals taken from CUDA events recorded on
those streams or the output of the lane simulator, in the SPEC's CSV shape
``op,stage,lane,start_s,end_s``.

The simulator (``stage_costs`` / ``simulate`` / ``simulate_backward``,
SPEC.md:570-597) is a FIFO list scheduler over the lanes {nvme, pcie, d2d,
compute}. ``costs_from_timeline`` turns a measured Timeline back into
per-op stage costs, so the simulator can be checked against the engine
(SURVEY §8 f4 "calibration against measured Timelines").
"""

from __future__ import annotations

from dataclasses import dataclass, field

STAGES = ("nc", "cg", "gg", "compute", "reduce_scatter", "grad_offload")
FETCH = ("nc", "cg", "gg")
LANES = {"nc": "nvme", "cg": "pcie", "gg": "d2d", "compute": "compute",
         "reduce_scatter": "d2d", "grad_offload": "pcie"}


@dataclass(frozen=True)
class Op:
    id: int
    param_keys: tuple
    param_bytes: int
    compute_flops: int


@dataclass(frozen=True)
class OperatorSequence:
    """Ordered ops {id, param keys, bytes, flops}; direction forward|backward."""
    ops: tuple
    direction: str = "forward"

    def __post_init__(self):
        ids = [o.id for o in self.ops]
        if self.direction == "forward" and ids != sorted(set(ids)):
            raise ValueError("forward op ids must be strictly increasing")

    def __len__(self):
        return len(self.ops)

    def reversed(self) -> "OperatorSequence":
        return OperatorSequence(tuple(reversed(self.ops)), "backward")


def trace_schedule(model_spec) -> tuple[OperatorSequence, OperatorSequence]:
    """forward sequence and the reversed backward sequence.

    ``model_spec`` is anything with ``operators()`` returning
    [(param_keys, param_bytes, flops)] in forward order — the toy
    ModelSpec of ``harness`` and the GPT engine both provide it. Tied /
    external keys appear in every consumer's fetch set. Re-tracing an
    unchanged spec yields an equal sequence (idempotent).
    """
    rows = list(model_spec.operators())
    if not rows:
        raise ValueError("empty model")
    ops = tuple(Op(i, tuple(keys), int(b), int(f)) for i, (keys, b, f) in enumerate(rows))
    for o in ops:
        if o.param_bytes <= 0 or o.compute_flops <= 0:
            raise ValueError("op bytes and flops must be positive")
    fwd = OperatorSequence(ops, "forward")
    return fwd, fwd.reversed()


@dataclass(frozen=True)
class PrefetchPlan:
    """Per executing slot: the ops whose nc / cg / gg stage to issue.

    ``slots[0]`` is the eager issue "at time 0" (before op 0 runs); slot i+1
    is issued when op i starts. Indices are positions in the sequence.
    """
    depths: tuple
    slots: tuple
    ops: tuple = ()      # op ids by position (Timeline labels)

    def issue(self, position: int) -> dict:
        return self.slots[position + 1]


def plan_prefetch(seq: OperatorSequence, depths=(3, 2, 1)) -> PrefetchPlan:
    """SPEC.md:560-568; matches oracle/schedule.py:plan_prefetch."""
    d_nc, d_cg, d_gg = depths
    if not (d_nc >= d_cg >= d_gg >= 1):
        raise ValueError("need d_nc >= d_cg >= d_gg >= 1")
    n = len(seq)
    eager = {"nc": list(range(min(n, d_nc))), "cg": list(range(min(n, d_cg))),
             "gg": list(range(min(n, d_gg)))}
    slots = [eager]
    for i in range(n):
        slot = {"nc": [], "cg": [], "gg": []}
        for stage, d in (("nc", d_nc), ("cg", d_cg), ("gg", d_gg)):
            if i + d < n:
                slot[stage].append(i + d)
        slots.append(slot)
    return PrefetchPlan(tuple(depths), tuple(slots), tuple(o.id for o in seq.ops))


@dataclass
class Timeline:
    """Intervals {op, stage, lane, start_s, end_s}.

    ``t0`` anchors ``total_s`` (simulated timelines start at 0 even when the
    first stages cost nothing and are not emitted); ``lanes`` overrides the
    stage -> lane map (see ``simulate_backward(lanes=...)``).
    """
    events: list = field(default_factory=list)
    t0: float | None = None
    lanes: dict | None = None

    def add(self, op: int, stage: str, start_s: float, end_s: float) -> None:
        self.events.append((op, stage, (self.lanes or LANES)[stage], start_s, end_s))

    @property
    def total_s(self) -> float:
        if not self.events:
            return 0.0
        start = self.t0 if self.t0 is not None else min(e[3] for e in self.events)
        return max(e[4] for e in self.events) - start

    @property
    def serial_s(self) -> float:
        return sum(e[4] - e[3] for e in self.events)

    def lane_busy_s(self, lane: str) -> float:
        """Union length of the intervals on one lane."""
        iv = sorted((e[3], e[4]) for e in self.events if e[2] == lane)
        tot, cur_s, cur_e = 0.0, None, None
        for s, e in iv:
            if cur_e is None or s > cur_e:
                if cur_e is not None:
                    tot += cur_e - cur_s
                cur_s, cur_e = s, e
            else:
                cur_e = max(cur_e, e)
        if cur_e is not None:
            tot += cur_e - cur_s
        return tot

    def hidden_fraction(self, transfer_lanes=("pcie", "d2d", "nvme")) -> float:
        """Share of transfer time overlapped with compute."""
        comp = sorted((e[3], e[4]) for e in self.events if e[2] == "compute")
        xfer = [(e[3], e[4]) for e in self.events if e[2] in transfer_lanes]
        tot = sum(e - s for s, e in xfer)
        if tot <= 0:
            return 1.0
        hid = 0.0
        for s, e in xfer:
            for cs, ce in comp:
                hid += max(0.0, min(e, ce) - max(s, cs))
        return min(1.0, hid / tot)

    def to_csv(self) -> str:
        lines = ["op,stage,lane,start_s,end_s"]
        for op, st, lane, s, e in self.events:
            lines.append(f"{op},{st},{lane},{s:.9f},{e:.9f}")
        return "\n".join(lines) + "\n"

    def summary(self) -> str:
        tot, ser = self.total_s, self.serial_s
        return f"total_s,serial_s,speedup\n{tot:.9f},{ser:.9f},{(ser / tot if tot else 1.0):.6f}\n"


# --------------------------------------------------------------------------- lane simulator
@dataclass(frozen=True)
class ClusterConfig:
    """The fields of SPEC.md:247-250. Defaults are the DGX-2-like profile of SPEC.md:319."""
    nodes: int = 1
    devices_per_node: int = 16
    device_mem_bytes: float = 32e9
    host_mem_bytes_per_node: float = 1.5e12
    nvme_bytes_per_node: float = 28e12
    pcie_bw_per_device: float = 12e9
    host_mem_bw_per_node: float = 48e9
    nvme_bw_per_node: float = 25e9
    device_device_bw: float = 300e9
    peak_tp_per_device: float = 70e12

    def __post_init__(self):
        for k in self.__dataclass_fields__:
            if not getattr(self, k) > 0:
                raise ValueError(f"{k} must be positive")

    @property
    def world_size(self) -> int:
        return self.nodes * self.devices_per_node

    @property
    def pcie_share(self) -> float:
        """Per-device host link: its own link, capped by the node's shared host bandwidth."""
        return min(self.pcie_bw_per_device, self.host_mem_bw_per_node / self.devices_per_node)

    @property
    def nvme_share(self) -> float:
        return self.nvme_bw_per_node / self.devices_per_node


def b200_cluster(nodes: int = 1, devices_per_node: int = 8, **override) -> ClusterConfig:
    """A B200 node profile built from this build's measurements.

    Sources per field:
    * pcie 55.6e9 B/s is the pinned H2D copy measured by ``bench.py`` (host_link_peak).
      Every GPU has its own x16 link, so the node total is ×devices.
    * NVMe 5.6e9 B/s is ``dd iflag=direct`` on the test box.
    * Peak 1422.7e12 is the sustained bf16 figure in MEASURED_PEAKS.json.
    * NVLink 5 at 900e9 B/s per direction is nominal, not measured (one GPU per box here).
    """
    vals = dict(nodes=nodes, devices_per_node=devices_per_node, device_mem_bytes=180e9,
                host_mem_bytes_per_node=196e9, nvme_bytes_per_node=256e9,
                pcie_bw_per_device=55.6e9, host_mem_bw_per_node=55.6e9 * devices_per_node,
                nvme_bw_per_node=5.6e9, device_device_bw=900e9, peak_tp_per_device=1422.7e12)
    vals.update(override)
    return ClusterConfig(**vals)


def stage_costs(cluster: ClusterConfig, tier_path: str, op: Op) -> dict:
    """Seconds per stage of one op; oracle/schedule.py:stage_costs.

    Transfer stage costs are bytes divided by the lane's bandwidth; compute is
    flops / peak_tp. The fetch path is nc (NVMe → host, the device's share of
    node NVMe bandwidth), then cg (host → device over its PCIe share), then gg
    (all-gather over the fabric, bytes·(W−1)/W). The backward adds
    reduce_scatter (the same fabric bytes) and grad_offload (the gradient shard
    back over PCIe; 0 when the tier path is the device).
    """
    if tier_path not in ("device", "host", "nvme"):
        raise ValueError(f"tier_path must be device|host|nvme, not {tier_path!r}")
    W = cluster.world_size
    shard = op.param_bytes / W
    fabric = op.param_bytes * (W - 1) / W / cluster.device_device_bw
    host = tier_path != "device"
    return {"nc": shard / cluster.nvme_share if tier_path == "nvme" else 0.0,
            "cg": shard / cluster.pcie_share if host else 0.0,
            "gg": fabric,
            "compute": op.compute_flops / cluster.peak_tp_per_device,
            "reduce_scatter": fabric,
            "grad_offload": shard / cluster.pcie_share if host else 0.0}


def _lane_key(stage: str, pos: int, depth: dict) -> tuple:
    """FIFO service order on a lane: (issue slot, phase, op position, stage order).

    A fetch stage of op j is issued in slot j − d (eagerly, slot −1, when j < d)
    at the start of that slot's compute. Compute runs in sequence order. The
    reduce-scatter and grad offload of op i are issued after compute(i)
    (phase 1). Sorting every item by this key is also a topological order of
    the dependency graph, so one sweep schedules everything.
    """
    k = STAGES.index(stage)
    if stage in FETCH:
        d = depth[stage]
        return (pos - d if pos >= d else -1, 0, pos, k)
    return (pos, 0 if stage == "compute" else 1, pos, k)


def _simulate(plan: PrefetchPlan, costs, stages, overlap: bool, lanes) -> Timeline:
    n = len(plan.slots) - 1
    if len(costs) != n:
        raise ValueError(f"{len(costs)} cost rows for a {n}-op plan")
    lanes = dict(LANES, **(lanes or {}))
    c = [[float(row.get(s, 0.0)) for s in stages] for row in costs]
    if any(x < 0 for row in c for x in row):
        raise ValueError("stage costs must be >= 0")
    ops = plan.ops or tuple(range(n))
    tl = Timeline(t0=0.0, lanes=lanes)
    if not overlap:   # every stage back to back in dependency order: total = sum
        t = 0.0
        for i in range(n):
            for s, x in zip(stages, c[i]):
                if x > 0:
                    tl.add(ops[i], s, t, t + x)
                t += x
        return tl
    depth = dict(zip(FETCH, plan.depths))
    items = sorted((_lane_key(s, i, depth), i, j, s) for i in range(n) for j, s in enumerate(stages))
    start, end, free = {}, {}, {}
    for key, i, j, s in items:
        t = free.get(lanes[s], 0.0)
        if j > 0:                                   # the op's previous stage
            t = max(t, end[i, stages[j - 1]])
        if s in FETCH and key[0] >= 0:              # issued when compute(slot) starts
            t = max(t, start[key[0], "compute"])
        start[i, s] = t
        end[i, s] = e = t + c[i][j]
        free[lanes[s]] = e
        if e > t:
            tl.add(ops[i], s, t, e)
    tl.events.sort(key=lambda ev: (ev[3], STAGES.index(ev[1]), ev[0]))
    return tl


def simulate(plan: PrefetchPlan, costs, overlap: bool = True, lanes: dict | None = None) -> Timeline:
    """Forward Timeline of a prefetch plan; oracle/schedule.py:simulate.

    ``costs[i]`` maps nc / cg / gg / compute to seconds for the op at sequence
    position i. With ``overlap=False`` the stages run back to back, so the
    total is the sum of all costs. Otherwise each lane serves its items FIFO
    in issue order, and an item starts once it is issued, its previous stage
    is done and its lane is free. Zero-cost stages are not emitted.
    """
    return _simulate(plan, costs, FETCH + ("compute",), overlap, lanes)


def simulate_backward(plan: PrefetchPlan, costs, overlap: bool = True,
                      lanes: dict | None = None) -> Timeline:
    """Backward Timeline: fetch → compute → reduce_scatter → grad_offload per op.

    rs(i+1) overlaps compute(i), and grad_offload(i+2) overlaps both, each on
    its own lane. ``plan`` is ``plan_prefetch`` of the backward sequence.
    ``lanes={"grad_offload": "pcie_d2h"}`` models a full-duplex host link.
    """
    return _simulate(plan, costs, STAGES, overlap, lanes)


def verify_timeline(tl: Timeline) -> None:
    """The validity check of SPEC.md:600: no lane overlap, stage order per op. Raises ValueError."""
    by_lane: dict = {}
    by_op: dict = {}
    for op, st, lane, s, e in tl.events:
        if e < s:
            raise ValueError(f"negative interval {op}/{st}")
        by_lane.setdefault(lane, []).append((s, e, op, st))
        by_op.setdefault(op, []).append((STAGES.index(st), s, e))
    for lane, iv in by_lane.items():
        iv.sort()
        for a, b in zip(iv, iv[1:]):
            if b[0] < a[1]:
                raise ValueError(f"lane {lane}: {a[2]}/{a[3]} overlaps {b[2]}/{b[3]}")
    for op, st in by_op.items():
        st.sort()
        for a, b in zip(st, st[1:]):
            if b[1] < a[2]:
                raise ValueError(f"op {op}: {STAGES[b[0]]} starts before {STAGES[a[0]]} ends")


def costs_from_timeline(tl: Timeline, ops, stage_map: dict | None = None) -> list:
    """Per-op stage costs measured on the engine (the union busy time of that op's spans).

    ``stage_map`` renames measured stages, e.g. {"cg": "grad_offload"} to
    count a bucket's optimizer-state H2D as host-link work after its compute.
    Returns one dict per entry of ``ops``, in order: the calibration input to
    ``simulate``.
    """
    stage_map = stage_map or {}
    spans: dict = {}
    for op, st, _lane, s, e in tl.events:
        spans.setdefault((op, stage_map.get(st, st)), []).append((s, e))
    out = []
    for op in ops:
        row = {}
        for st in STAGES:
            iv = sorted(spans.get((op, st), ()))
            tot, cs, ce = 0.0, None, None
            for s, e in iv:
                if ce is None or s > ce:
                    if ce is not None:
                        tot += ce - cs
                    cs, ce = s, e
                else:
                    ce = max(ce, e)
            if ce is not None:
                tot += ce - cs
            row[st] = tot
        out.append(row)
    return out
