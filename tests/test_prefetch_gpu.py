"""The prefetch plan drives the engine's fetches (PAPER §6.2).

With params off HBM every fetch position p runs three stages: nc (NVMe -> pinned, store
workers), cg (pinned -> HBM staging, the H2D stream) and gg (staging -> gathered slot).
While position p runs the engine issues nc(p + 3), cg(p + 2), gg(p + 1) — the plan's
issue sets — and a prefetch byte budget delays early stages without changing results.
Every placement trains bit for bit like the all-HBM engine (the step is deterministic).
"""

import numpy as np
import pytest
import torch

from paper_2104_07857_b200 import gpt as eg
from paper_2104_07857_b200.comm import LocalComm
from paper_2104_07857_b200.gpt import Placement
from paper_2104_07857_b200.store import TierKind

pytestmark = pytest.mark.gpu

CFG = eg.GPTConfig(nl=4, hd=128, heads=2, seq=128, vocab=256, batch=2)
D, H, V = TierKind.DEVICE, TierKind.HOST, TierKind.NVME


def run(placement, steps=3, world=2, **kw):
    eng = eg.GPTZeroEngine(CFG, LocalComm(world), lr=1e-3, placement=placement,
                           offload_chunk=20_000, **kw)
    losses = [eng.step([eg.synthetic_tokens(CFG, 7, r, s) for r in range(world)]).item()
              for s in range(steps)]
    torch.cuda.synchronize()
    return eng, losses


def same_states(a, b, world=2):
    for key in a.by_key:
        for r in range(world):
            sa, sb = a.shard(key, r), b.shard(key, r)
            for n in ("p32", "m", "v"):
                assert torch.equal(sa[n].cpu().view(torch.int32), sb[n].cpu().view(torch.int32)), (key, r, n)
            assert torch.equal(sa["p16"].cpu().view(torch.int16), sb["p16"].cpu().view(torch.int16))


@pytest.mark.parametrize("params,optim", [(H, D), (H, H), (V, H)])
def test_offloaded_params_train_like_hbm(params, optim, tmp_path):
    ref, lr = run(Placement(D, D))
    eng, le = run(Placement(params, optim), nvme_root=str(tmp_path))
    assert le == lr
    same_states(ref, eng)
    if params is V:     # the shard files hold the updated bf16 params
        for key in eng.by_key:
            for li in range(2):
                assert torch.equal(eng.param_file_shard(key, li).view(torch.int16),
                                   eng.shard(key, li)["p16"].cpu().view(torch.int16))
        eng.close()


def positions(eng, stage):
    return {q: at for at, st, q in eng.issue_log if st == stage}


@pytest.mark.parametrize("params", [H, V])
def test_plan_depths_are_executed(params, tmp_path):
    """depths (3, 2, 1): the cg of position q is issued while q - 2 runs (the first two
    eagerly at step start), the nc (NVMe) while q - 3 runs; every stage precedes its
    successor; the step's fetch list covers forward, head and the backward re-gathers."""
    eng, _ = run(Placement(params, H), steps=2, nvme_root=str(tmp_path))
    n = len(eng._flist)
    assert n == 1 + CFG.nl + 1 + (CFG.nl - 1) and eng._fpos == n
    cg = positions(eng, "cg")
    assert sorted(cg) == list(range(n))
    for q in range(n):      # plan.issue(q - 2) runs as fetch position q - 1 starts
        assert cg[q] == (0 if q < 2 else q - 1), (q, cg[q])
    if params is V:
        nc = positions(eng, "nc")
        assert sorted(nc) == list(range(n))
        for q in range(n):
            assert nc[q] == (0 if q < 3 else q - 2), (q, nc[q])
            assert nc[q] <= cg[q]
        eng.close()


def test_budget_delays_but_does_not_change_results(tmp_path):
    """A byte budget of one bucket: no stage runs ahead of its successor's need (cg of q
    at q itself), yet the training is the same."""
    ref, lr = run(Placement(H, H), steps=2)
    one = max(b.shard for b in ref.buckets) * 2 * 2
    eng, le = run(Placement(H, H), steps=2, prefetch_budget=one)
    assert le == lr
    same_states(ref, eng)
    cg = positions(eng, "cg")
    assert any(cg[q] == q for q in cg)       # forced just in time
    ej, _ = run(Placement(H, H), steps=2, prefetch_depths=(1, 1, 1))
    assert all(at == q for q, at in positions(ej, "cg").items())   # depths (1,1,1): JIT


def test_plan_matches_schedule_plan():
    """The engine's per-step plan is schedule.plan_prefetch over its fetch list."""
    from paper_2104_07857_b200.schedule import plan_prefetch
    eng, _ = run(Placement(H, D), steps=1)
    plan = eng._fplan
    assert plan.depths == (3, 2, 1)
    assert plan.slots[0] == {"nc": [0, 1, 2], "cg": [0, 1], "gg": [0]}
    assert plan.issue(0) == {"nc": [3], "cg": [2], "gg": [1]}
    assert len(plan.slots) == len(eng._flist) + 1
    assert eng.plan == plan_prefetch(eng.fwd_seq, (3, 2, 1))
