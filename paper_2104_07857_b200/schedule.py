"""Overlap-centric schedule: operator trace, prefetch plan, measured Timeline.

``trace_schedule`` records the operator sequence (PAPER §6.2 "constructing
an internal map of the operator sequence"); ``plan_prefetch`` decides, for
every op i, which later ops' fetch stages to issue while i runs — nc for
i+d_nc, cg for i+d_cg, gg for i+d_gg, default depths (3, 2, 1)
(SPEC.md:560-568). The engine executes the plan on side CUDA streams:

    nc  NVMe -> pinned host        (store worker threads)
    cg  pinned host -> HBM         (H2D copy-engine stream)
    gg  HBM shards -> full params  (gather stream: NVLink all-gather / P2P)

``Timeline`` holds real intervals taken from CUDA events recorded on those
streams, in the SPEC's CSV shape ``op,stage,lane,start_s,end_s``
(SPEC.md:544-547, 615); the simulator of SPEC.md:570-597 is not part of
this build (analytic, out of scope).
"""

from __future__ import annotations

from dataclasses import dataclass, field

STAGES = ("nc", "cg", "gg", "compute", "reduce_scatter", "grad_offload")
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
    return PrefetchPlan(tuple(depths), tuple(slots))


@dataclass
class Timeline:
    """Measured intervals {op, stage, lane, start_s, end_s}."""
    events: list = field(default_factory=list)

    def add(self, op: int, stage: str, start_s: float, end_s: float) -> None:
        self.events.append((op, stage, LANES[stage], start_s, end_s))

    @property
    def total_s(self) -> float:
        if not self.events:
            return 0.0
        return max(e[4] for e in self.events) - min(e[3] for e in self.events)

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
