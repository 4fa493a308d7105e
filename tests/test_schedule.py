"""Operator trace, prefetch plan and Timeline (CPU): the product schedule equals the oracle's."""

import pytest

from oracle.schedule import plan_prefetch as o_plan
from paper_2104_07857_b200 import harness as H
from paper_2104_07857_b200.schedule import Timeline, plan_prefetch, trace_schedule


def toy(tied=False):
    L = H.LayerSpec
    layers = [L("linear", 8, 16, "relu"), L("linear", 16, 16, "relu"), L("linear", 16, 16),
              L("linear", 16, 4)]
    return H.ModelSpec(layers, tied_pairs=[(1, 2)] if tied else [], seed=7)


def test_trace_forward_backward():
    fwd, bwd = trace_schedule(toy())
    assert [o.id for o in fwd.ops] == [0, 1, 2, 3]
    assert [o.id for o in bwd.ops] == [3, 2, 1, 0]
    assert trace_schedule(toy()) == (fwd, bwd)          # re-trace idempotent


def test_tied_key_in_both_consumers():
    fwd, _ = trace_schedule(toy(tied=True))
    assert fwd.ops[1].param_keys == fwd.ops[2].param_keys == ("layer1",)


def test_empty_model_rejected():
    class Empty:
        def operators(self):
            return []
    with pytest.raises(ValueError):
        trace_schedule(Empty())


@pytest.mark.parametrize("n,depths", [(5, (3, 2, 1)), (1, (3, 2, 1)), (7, (1, 1, 1)), (4, (4, 2, 2))])
def test_plan_matches_oracle(n, depths):
    class Spec:
        def operators(self):
            return [(("k%d" % i,), 10, 10) for i in range(n)]
    fwd, _ = trace_schedule(Spec())
    plan = plan_prefetch(fwd, depths)
    ref = o_plan(n, depths)
    for slot, oslot in zip(plan.slots, ref):
        assert {k: slot[k] for k in ("nc", "cg", "gg")} == {k: oslot[k] for k in ("nc", "cg", "gg")}
    if n == 5 and depths == (3, 2, 1):
        assert plan.issue(0) == {"nc": [3], "cg": [2], "gg": [1]}


def test_invalid_depths():
    fwd, _ = trace_schedule(toy())
    with pytest.raises(ValueError):
        plan_prefetch(fwd, (1, 2, 1))


def test_timeline_csv_and_hidden_fraction():
    tl = Timeline()
    tl.add(0, "compute", 0.0, 1.0)
    tl.add(1, "gg", 0.5, 1.5)      # half hidden behind op 0's compute
    tl.add(1, "compute", 1.5, 2.5)
    assert tl.total_s == 2.5 and tl.serial_s == 3.0
    assert abs(tl.hidden_fraction() - 0.5) < 1e-12
    assert tl.to_csv().splitlines()[0] == "op,stage,lane,start_s,end_s"
    assert tl.summary().splitlines()[0] == "total_s,serial_s,speedup"
    assert abs(tl.lane_busy_s("compute") - 2.0) < 1e-12
