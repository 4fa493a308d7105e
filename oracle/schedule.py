"""CPU restatement of the overlap-engine's tracer and prefetch planner.

TEST INFRASTRUCTURE (see oracle/__init__.py). ``trace_schedule`` and
``plan_prefetch`` are on the executed path. The lane simulator (``stage_costs``,
``simulate``) is restated here as a brute-force fixed point
over its constraints, independent of the product's single topological sweep.
"""

STAGES = ("nc", "cg", "gg", "compute", "reduce_scatter", "grad_offload")
LANE = {"nc": "nvme", "cg": "pcie", "gg": "d2d", "compute": "compute",
        "reduce_scatter": "d2d", "grad_offload": "pcie"}


def stage_costs(cluster: dict, tier_path: str, param_bytes: int, flops: float) -> dict:
    """SPEC.md:570-578. ``cluster`` holds the SPEC.md:248 field names.

    nc: the device's NVMe share (node bandwidth / devices per node).
    cg: the device's PCIe share, min(own link, node host bandwidth / devices).
    gg / reduce_scatter: all-gather bytes·(W−1)/W over the device fabric.
    grad_offload: the gradient shard over PCIe.
    """
    W = cluster["nodes"] * cluster["devices_per_node"]
    pcie = min(cluster["pcie_bw_per_device"],
               cluster["host_mem_bw_per_node"] / cluster["devices_per_node"])
    nvme = cluster["nvme_bw_per_node"] / cluster["devices_per_node"]
    shard = param_bytes / W
    ag = param_bytes * (W - 1) / W / cluster["device_device_bw"]
    return {"nc": shard / nvme if tier_path == "nvme" else 0.0,
            "cg": shard / pcie if tier_path in ("host", "nvme") else 0.0,
            "gg": ag, "compute": flops / cluster["peak_tp_per_device"],
            "reduce_scatter": ag,
            "grad_offload": shard / pcie if tier_path in ("host", "nvme") else 0.0}


def simulate(depths, costs: list[dict], backward: bool = False, overlap: bool = True,
             lanes: dict | None = None):
    """SPEC.md:580-597 as a constraint system, solved by iterating to a fixed point.

    Items are (position i, stage). Each start is the max of:
    * the end of the op's previous stage (nc → cg → gg → compute → rs → offload);
    * for a fetch stage of op j at depth d with j ≥ d: the start of compute(j − d),
      the slot that issues it;
    * the end of the item served before it on its lane.
    Lane service is FIFO in issue order (slot, then post-compute items, then
    position, then stage order); eager fetches are slot −1.
    Returns (events [(i, stage, lane, start, end)] for positive costs, total).
    """
    stages = STAGES if backward else STAGES[:4]
    lane = dict(LANE, **(lanes or {}))
    n = len(costs)
    cost = {(i, s): float(costs[i].get(s, 0.0)) for i in range(n) for s in stages}
    if not overlap:
        ev, t = [], 0.0
        for i in range(n):
            for s in stages:
                if cost[i, s] > 0:
                    ev.append((i, s, lane[s], t, t + cost[i, s]))
                t += cost[i, s]
        return ev, t
    d = dict(zip(("nc", "cg", "gg"), depths))

    def issue(i, s):
        if s in d:
            return (i - d[s] if i >= d[s] else -1, 0, i, STAGES.index(s))
        return (i, 0 if s == "compute" else 1, i, STAGES.index(s))
    order = {}
    for i in range(n):
        for s in stages:
            order.setdefault(lane[s], []).append((issue(i, s), i, s))
    before = {}
    for items in order.values():
        items.sort()
        for a, b in zip(items, items[1:]):
            before[b[1], b[2]] = (a[1], a[2])
    start = {k: 0.0 for k in cost}
    for _ in range(len(cost) + 1):
        changed = False
        for (i, s) in cost:
            t = 0.0
            k = stages.index(s)
            if k > 0:
                p = (i, stages[k - 1])
                t = max(t, start[p] + cost[p])
            if s in d and i >= d[s]:
                t = max(t, start[i - d[s], "compute"])
            if (i, s) in before:
                p = before[i, s]
                t = max(t, start[p] + cost[p])
            if t != start[i, s]:
                start[i, s], changed = t, True
        if not changed:
            break
    else:
        raise RuntimeError("dependency cycle")
    ev = sorted(((i, s, lane[s], start[i, s], start[i, s] + cost[i, s])
                 for (i, s) in cost if cost[i, s] > 0), key=lambda e: (e[3], STAGES.index(e[1]), e[0]))
    total = max((start[k] + cost[k] for k in cost), default=0.0)
    return ev, total


def trace_forward_backward(op_param_keys: list[tuple[str, ...]]):
    """Forward ids [0..L-1] and reversed backward ids."""
    if not op_param_keys:
        raise ValueError("empty model")
    fwd = list(range(len(op_param_keys)))
    return fwd, list(reversed(fwd))


def plan_prefetch(n_ops: int, depths=(3, 2, 1)) -> list[dict]:
    """while executing op i issue nc(i+d_nc), cg(i+d_cg), gg(i+d_gg).

    Ops within ``depth`` of the start are issued eagerly "at time 0" in
    dependency order — recorded here as the issue list of a virtual slot -1.
    Returns one dict per slot (-1 .. n_ops-1): {"at": i, "nc": [...], "cg": [...], "gg": [...]}.
    """
    d_nc, d_cg, d_gg = depths
    if not (d_nc >= d_cg >= d_gg >= 1):
        raise ValueError("need d_nc >= d_cg >= d_gg >= 1")
    plan = []
    eager = {"at": -1, "nc": [], "cg": [], "gg": []}
    for j in range(min(n_ops, d_nc)):
        eager["nc"].append(j)
    for j in range(min(n_ops, d_cg)):
        eager["cg"].append(j)
    for j in range(min(n_ops, d_gg)):
        eager["gg"].append(j)
    plan.append(eager)
    for i in range(n_ops):
        slot = {"at": i, "nc": [], "cg": [], "gg": []}
        for stage, d in (("nc", d_nc), ("cg", d_cg), ("gg", d_gg)):
            j = i + d
            if j < n_ops:
                slot[stage].append(j)
        plan.append(slot)
    return plan
