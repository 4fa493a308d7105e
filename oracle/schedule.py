"""CPU restatement of the overlap-engine's tracer and prefetch planner.

TEST INFRASTRUCTURE (see oracle/__init__.py). Only ``trace_schedule`` and
``plan_prefetch`` are on the executed path; the lane simulator
(``stage_costs`` / ``simulate``) is analytic and out of scope.
"""

from __future__ import annotations


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
