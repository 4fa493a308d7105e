"""Lane simulator on CPU: the SPEC examples, the invariants of
SPEC.md:599-603 as properties, and the product's sweep equal to the oracle's fixed point."""

import dataclasses
import random

import pytest
from hypothesis import given, settings, strategies as st

from oracle import schedule as O
from paper_2104_07857_b200 import schedule as S


def seq_of(n, nbytes=1 << 20, flops=1e9):
    return S.OperatorSequence(tuple(S.Op(i, (f"l{i}",), nbytes, flops) for i in range(n)))


def plan(n, depths=(3, 2, 1), backward=False):
    seq = seq_of(n)
    return S.plan_prefetch(seq.reversed() if backward else seq, depths)


def rand_costs(rng, n, zero_p=0.2):
    return [{s: (0.0 if rng.random() < zero_p else rng.uniform(0.1, 3.0)) for s in S.STAGES}
            for _ in range(n)]


def oracle_cluster(c: S.ClusterConfig) -> dict:
    return dataclasses.asdict(c)


# -- stage_costs -------------------------------------------------------------------------
def test_stage_costs_examples():
    c = S.ClusterConfig()
    op = S.Op(0, ("w",), (64 << 20) * c.world_size, 1e12)
    cost = S.stage_costs(c, "nvme", op)
    assert cost["nc"] == pytest.approx(0.042, abs=1.5e-3)
    assert S.stage_costs(c, "host", op)["nc"] == 0.0
    dev = S.stage_costs(c, "device", op)
    assert dev["nc"] == dev["cg"] == dev["grad_offload"] == 0.0
    op2 = S.Op(0, ("w",), op.param_bytes * 2, op.compute_flops)
    c2 = S.stage_costs(c, "nvme", op2)
    for s in ("nc", "cg", "gg", "reduce_scatter", "grad_offload"):  # linearity
        assert c2[s] == 2 * cost[s]
    assert cost == O.stage_costs(oracle_cluster(c), "nvme", op.param_bytes, op.compute_flops)
    assert S.stage_costs(c, "nvme", op)["cg"] == pytest.approx((64 << 20) / 3e9)   # 48e9/16 share


def test_stage_costs_rejects_bad_input():
    with pytest.raises(ValueError):
        S.stage_costs(S.ClusterConfig(), "tape", S.Op(0, (), 1, 1))
    with pytest.raises(ValueError):
        S.ClusterConfig(pcie_bw_per_device=0)
    b = S.b200_cluster()
    assert b.world_size == 8 and b.pcie_share == 55.6e9


# -- simulate: SPEC examples ----------------------------------------------------------------
def test_serial_total_is_sum():
    rng = random.Random(1)
    costs = rand_costs(rng, 6)
    tl = S.simulate(plan(6), costs, overlap=False)
    assert tl.total_s == pytest.approx(sum(c[s] for c in costs for s in S.STAGES[:4]))
    assert tl.summary().splitlines()[1].endswith(",1.000000")
    S.verify_timeline(tl)


@pytest.mark.parametrize("n", [1, 2, 5, 40])
def test_equal_costs_pipeline(n):
    c = 0.5
    costs = [{"nc": c, "cg": c, "gg": c, "compute": c}] * n
    tl = S.simulate(plan(n), costs)
    assert tl.total_s == pytest.approx((n + 3) * c)
    assert S.simulate(plan(n), costs, overlap=False).total_s == pytest.approx(4 * n * c)
    S.verify_timeline(tl)


def test_zero_transfer_is_sum_of_compute():
    costs = [{"compute": x} for x in (1.0, 2.0, 0.5)]
    assert S.simulate(plan(3), costs).total_s == 3.5
    b = S.simulate_backward(plan(3, backward=True), costs)
    assert b.total_s == 3.5


def test_device_tier_has_empty_nc_cg_lanes():
    c = S.b200_cluster()
    seq = seq_of(6, 100 << 20, 2e12)
    costs = [S.stage_costs(c, "device", o) for o in seq.ops]
    tl = S.simulate(S.plan_prefetch(seq), costs)
    assert tl.lane_busy_s("nvme") == tl.lane_busy_s("pcie") == 0.0
    assert tl.lane_busy_s("d2d") > 0


def test_balanced_backward_steady_state():
    n, c = 60, 1.0
    costs = [{s: c for s in S.STAGES}] * n
    tl = S.simulate_backward(plan(n, backward=True), costs)
    # pcie carries cg + grad_offload and d2d gg + reduce_scatter (2c per op each):
    # steady state = the busiest lane's cost per op
    per_op = (tl.total_s - S.simulate_backward(plan(n // 2, backward=True),
                                               costs[:n // 2]).total_s) / (n - n // 2)
    assert per_op == pytest.approx(2 * c)
    duplex = {"grad_offload": "pcie_d2h", "reduce_scatter": "d2d_rs"}
    tl2 = S.simulate_backward(plan(n, backward=True), costs, lanes=duplex)
    per_op2 = (tl2.total_s - S.simulate_backward(plan(n // 2, backward=True), costs[:n // 2],
                                                 lanes=duplex).total_s) / (n - n // 2)
    assert per_op2 == pytest.approx(c)                             # every lane c per op
    S.verify_timeline(tl2)


def test_eager_issue_order():
    tl = S.simulate(plan(1), [{"nc": 1, "cg": 1, "gg": 1, "compute": 1}])
    assert [(e[1], e[3]) for e in tl.events] == [("nc", 0), ("cg", 1), ("gg", 2), ("compute", 3)]


def test_cost_rows_must_match_plan():
    with pytest.raises(ValueError):
        S.simulate(plan(3), [{"compute": 1}] * 2)
    with pytest.raises(ValueError):
        S.simulate(plan(1), [{"compute": -1}])


def test_verifier_catches_overlap():
    tl = S.Timeline(t0=0.0)
    tl.add(0, "cg", 0.0, 2.0)
    tl.add(1, "cg", 1.0, 3.0)
    with pytest.raises(ValueError):
        S.verify_timeline(tl)
    tl = S.Timeline(t0=0.0)
    tl.add(0, "gg", 0.0, 2.0)
    tl.add(0, "compute", 1.0, 3.0)
    with pytest.raises(ValueError):
        S.verify_timeline(tl)


# -- properties and oracle agreement ----------------------------------------
depths_st = st.tuples(st.integers(1, 4), st.integers(1, 4), st.integers(1, 4)).map(
    lambda t: tuple(sorted(t, reverse=True)))


@settings(max_examples=300, deadline=None)
@given(n=st.integers(1, 12), depths=depths_st, seed=st.integers(0, 10 ** 6),
       backward=st.booleans(), duplex=st.booleans())
def test_properties_and_oracle(n, depths, seed, backward, duplex):
    rng = random.Random(seed)
    costs = rand_costs(rng, n)
    lanes = {"grad_offload": "pcie_d2h"} if duplex else None
    p = plan(n, depths, backward)
    run = S.simulate_backward if backward else S.simulate
    stages = S.STAGES if backward else S.STAGES[:4]
    tl = run(p, costs, lanes=lanes)
    S.verify_timeline(tl)
    ev, total = O.simulate(depths, costs, backward=backward, lanes=lanes)
    assert tl.total_s == total                                     # bit-identical
    ids = p.ops
    assert sorted(tl.events) == sorted((ids[i], s, ln, a, b) for i, s, ln, a, b in ev)
    serial = run(p, costs, overlap=False, lanes=lanes)
    assert tl.total_s <= serial.total_s + 1e-12                    # overlapped <= serial
    lane_sum = {}
    for i in range(n):
        for s in stages:
            ln = (lanes or {}).get(s, S.LANES[s])
            lane_sum[ln] = lane_sum.get(ln, 0.0) + costs[i][s]
    assert tl.total_s >= max(lane_sum.values()) - 1e-12            # lane lower bound
    i, s = rng.randrange(n), rng.choice(stages)                    # monotone in every cost
    bumped = [dict(c) for c in costs]
    bumped[i][s] += rng.uniform(0.01, 2.0)
    assert run(p, bumped, lanes=lanes).total_s >= tl.total_s


def test_backward_never_slower_than_serial_1000_trials():
    rng = random.Random(7)
    for _ in range(1000):
        n = rng.randint(1, 10)
        costs = rand_costs(rng, n, zero_p=0.1)
        p = plan(n, backward=True)
        assert (S.simulate_backward(p, costs).total_s
                <= S.simulate_backward(p, costs, overlap=False).total_s + 1e-12)


def test_speedup_approaches_four():
    for n, lo in ((10, 3.0), (100, 3.8), (1000, 3.98)):
        costs = [{"nc": 1, "cg": 1, "gg": 1, "compute": 1}] * n
        tl = S.simulate(plan(n), costs)
        assert tl.serial_s / tl.total_s >= lo


# -- calibration ------------------------------------------------------------------------------
def test_costs_from_timeline_roundtrip():
    rng = random.Random(3)
    costs = rand_costs(rng, 5, zero_p=0.0)
    p = plan(5, backward=True)
    tl = S.simulate_backward(p, costs, lanes={"grad_offload": "pcie_d2h"})
    back = S.costs_from_timeline(tl, p.ops)
    for a, b in zip(costs, back):
        for s in S.STAGES:
            assert b[s] == pytest.approx(a[s])
    again = S.simulate_backward(p, back, lanes={"grad_offload": "pcie_d2h"})
    assert again.total_s == pytest.approx(tl.total_s)
    merged = S.costs_from_timeline(tl, p.ops, stage_map={"reduce_scatter": "grad_offload"})
    assert merged[0]["reduce_scatter"] == 0.0
