"""The partitioned GPT step on the GPU against the CPU oracle (oracle/gpt.py).

Layout and init are bit-exact. The step (BASELINE config 1 at world 2, 3 steps; a
1.3B-shape block; ragged worlds) is checked per step on the loss, every gradient
shard and the Adam update of every master element, with tolerances set at ~5x the
error measured on B200 (TOL_BF16 / TOL_FP32 below, scripts/parity_probe.py): tight
enough that a skipped, doubled or misrouted update fails.
"""

import numpy as np
import pytest
import torch

from oracle import gpt as og
from oracle import numerics as nx
from paper_2104_07857_b200 import gpt as eg
from paper_2104_07857_b200.comm import LocalComm

pytestmark = pytest.mark.gpu

SMALL = eg.GPTConfig(nl=2, hd=128, heads=2, seq=128, vocab=256, batch=2)


def ocfg(c):
    return og.GPTConfig(c.nl, c.hd, c.heads, c.seq, c.vocab, c.batch)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def batches_for(c, world, step=0):
    return [eg.synthetic_tokens(c, 7, r, step) for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("half,kind", [(torch.bfloat16, nx.HALF_BF16), (torch.float16, nx.HALF_FP16)])
def test_init_layout_bit_exact(world, half, kind):
    eng = eg.GPTZeroEngine(SMALL, LocalComm(world), half_dtype=half)
    st = og.init_partitioned(ocfg(SMALL), world, half_kind=kind)
    for key in st.p16:
        for r in range(world):
            s = eng.shard(key, r)
            assert np.array_equal(s["p32"].cpu().numpy(), st.p32[key][r]), (key, r)
            got = s["p16"].cpu().view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(got, st.p16[key][r]), (key, r)
            assert not s["m"].any() and not s["v"].any()
        full = eng.gathered(key).cpu().view(torch.int16).numpy().view(np.uint16)
        want = nx.f32_to_half_bits(og.init_bucket_range(7, eng.by_key[key].op,
                                                        og.buckets(ocfg(SMALL))[eng.by_key[key].op][2],
                                                        0, st.full_len[key]), kind)
        assert np.array_equal(full, want)


def update_errors(eng, prev, st, lr):
    """Adam update of the GPU step vs the oracle's, per element in units of lr:
    (fraction of elements off by more than 0.1*lr, relative L2 of the update difference).
    A skipped or wrong update is off by ~lr on most elements: fraction ~1, rel ~1."""
    errs, num, den = [], 0.0, 0.0
    for key in st.p32:
        for r in range(st.world):
            p = eng.shard(key, r)["p32"].cpu().numpy().astype(np.float64)
            dg = p - prev[key][r]
            do = st.p32[key][r].astype(np.float64) - prev[key][r]
            errs.append(np.abs(dg - do) / lr)
            num += float(((dg - do) ** 2).sum())
            den += float((do ** 2).sum())
    e = np.concatenate(errs)
    return float((e > 0.1).mean()), float(np.sqrt(num / den))


def run_vs_oracle(cfg, world, steps, lr, tol, half=torch.bfloat16, compute=None, **kw):
    """``steps`` partitioned steps of the engine and the CPU oracle on the same seeded
    tokens, checked per step against ``tol`` = (loss rel, grad-shard rel L2,
    fraction of update elements off by > 0.1 lr, update rel L2)."""
    kind = nx.HALF_BF16 if half == torch.bfloat16 else nx.HALF_FP16
    eng = eg.GPTZeroEngine(cfg, LocalComm(world), lr=lr, half_dtype=half, compute_dtype=compute, **kw)
    eng.capture_grads = True
    st = og.init_partitioned(ocfg(cfg), world, half_kind=kind)
    for step in range(steps):
        prev = {k: [s.astype(np.float64) for s in st.p32[k]] for k in st.p32}
        bs = batches_for(cfg, world, step)
        loss = eng.step(bs).item()
        oloss, gsh = og.train_step(st, [(t.cpu().numpy(), y.cpu().numpy()) for t, y in bs], lr=lr)
        assert abs(loss - oloss) <= tol[0] * abs(oloss), (step, loss, oloss)
        for key in gsh:
            for r in range(world):
                e = rel(eng.grad_shards[key][r].cpu().numpy(), gsh[key][r])
                assert e < tol[1], (step, key, r, e)
        frac, urel = update_errors(eng, prev, st, lr)
        assert frac < tol[2] and urel < tol[3], (step, frac, urel)
    return eng, st


# Tolerances ~5x the errors measured on B200 (scripts/parity_probe.py; per step, worst of
# 3): bf16 compute vs the fp32 oracle: loss 4.4e-5, grad shards 1.1e-2, update elements
# off by > 0.1 lr 1.2 %, update rel L2 0.21. fp32 compute (fp16 params): loss 7.5e-8,
# grads 1.8e-4, 2.4e-6, 2.1e-3. A skipped or wrong Adam update gives ~1 and ~1.
TOL_BF16 = (2e-4, 5e-2, 5e-2, 0.5)
TOL_FP32 = (1e-6, 1e-3, 1e-4, 1e-2)


@pytest.mark.parametrize("act_ckpt", [None, "host"])
def test_config1_bf16_matches_oracle(act_ckpt):
    """BASELINE config 1 (nl4 / hd256 / 4 heads / seq128 / batch4 / V512), world 2, 3 steps
    against the CPU oracle; with act_ckpt="host" the block inputs go to pinned host DRAM
    and the backward recomputes from them (PAPER §5.1.2) — checked against the oracle
    directly, not against the no-checkpoint engine."""
    eng, _ = run_vs_oracle(eg.TINY, 2, 3, 1e-3, TOL_BF16, act_ckpt=act_ckpt)
    if act_ckpt == "host":
        assert eng.ckpt_bytes > 0


def test_config1_fp32_compute_matches_oracle():
    """fp32 compute (half params widened) against the fp32 oracle: the
    remaining error is summation order and single-ulp flips of the fp16 gradient
    contributions."""
    torch.backends.cuda.matmul.allow_tf32 = False
    run_vs_oracle(eg.TINY, 2, 3, 1e-3, TOL_FP32, half=torch.float16, compute=torch.float32)


@pytest.mark.parametrize("world", [1, 3])
def test_small_worlds_match_oracle(world):
    """Ragged world sizes (zero-padded shards) on the small config."""
    run_vs_oracle(SMALL, world, 2, 1e-3, TOL_BF16)


def test_1p3b_block_shape_matches_oracle():
    """One step of a block at the BASELINE 1.3B shape (hd 2048, 16 heads, seq 1024,
    V 50304, one sequence). Measured: loss 1.6e-5, grads 6.2e-3, 0.25 %, 0.058."""
    c = eg.GPTConfig(nl=1, hd=2048, heads=16, seq=1024, vocab=50304, batch=1)
    run_vs_oracle(c, 1, 1, 1e-4, (1e-4, 3e-2, 2e-2, 0.25))


def test_two_q_tile_attention_steps_match_oracle():
    """S = 256 runs the two-Q-tile attention forward (and the TMEM-resident P^T / dS^T / dS
    backward) inside the step: 3 partitioned steps at world 2 against the oracle."""
    c = eg.GPTConfig(nl=2, hd=256, heads=2, seq=256, vocab=512, batch=2)
    run_vs_oracle(c, 2, 3, 1e-3, TOL_BF16)


@pytest.mark.parametrize("world", [1, 2])
def test_cuda_graph_step_matches_eager(world):
    """The captured step replays the same math: device Adam counter + static inputs."""
    a = eg.GPTZeroEngine(SMALL, LocalComm(world), lr=1e-3)
    b = eg.GPTZeroEngine(SMALL, LocalComm(world), lr=1e-3)
    la, lb = [], []
    for step in range(5):
        bs = batches_for(SMALL, world, step)
        la.append(a.step(bs).item())
        lb.append(b.step_graphed(bs).item())
    assert la == lb                       # bitwise: replay == eager
    assert int(a.adam.step.item()) == int(b.adam.step.item()) == 5
    for key in a.by_key:
        torch.testing.assert_close(a.shard(key, 0)["p32"], b.shard(key, 0)["p32"], rtol=0, atol=0)


def test_device_adam_constants_match_host_folding():
    from paper_2104_07857_b200 import _lib, kernels
    st = kernels.DeviceAdamState(3e-4, (0.9, 0.95), 1e-8)
    for t in range(1, 200):
        st.advance()
        h = _lib.adam_consts(3e-4, 0.9, 0.95, 1e-8, t)
        want = np.array([h.lr, h.b1, h.omb1, h.b2, h.omb2, h.bc1, h.bc2, h.eps], np.float32)
        assert np.array_equal(st.consts.cpu().numpy(), want), t


@pytest.mark.parametrize("mode", ["device", "host"])
def test_activation_checkpointing_matches(mode):
    """Recompute from checkpoints (kept in HBM or offloaded to pinned host) gives the
    same step as keeping every activation."""
    a = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3)
    b = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, act_ckpt=mode, trace=(mode == "host"))
    for step in range(3):
        bs = batches_for(SMALL, 2, step)
        la, lb = a.step(bs).item(), b.step(bs).item()
        assert la == lb, (step, la, lb)
    for key in a.by_key:
        torch.testing.assert_close(a.shard(key, 1)["p32"], b.shard(key, 1)["p32"], rtol=0, atol=0)
    if mode == "host":
        assert b.ckpt_bytes > 0
        stages = {e[1] for e in b.timeline().events}
        assert {"cg", "grad_offload", "compute"} <= stages


@pytest.mark.parametrize("hd,heads", [(4096, 32), (8192, 64)])
def test_10b_70b_layer_shapes(hd, heads):
    """One block at the 10B / 70B widths (BASELINE configs 3 and 5): the libzinf path
    agrees with the torch-op path."""
    c = eg.GPTConfig(nl=1, hd=hd, heads=heads, seq=128, vocab=512, batch=1)
    a = eg.GPTZeroEngine(c, LocalComm(1), lr=1e-4, fused=True)
    la = a.step([eg.synthetic_tokens(c, 7, 0)]).item()
    del a
    torch.cuda.empty_cache()
    b = eg.GPTZeroEngine(c, LocalComm(1), lr=1e-4, fused=False)
    lb = b.step([eg.synthetic_tokens(c, 7, 0)]).item()
    assert np.isfinite(la) and abs(la - lb) <= 2e-3 * abs(lb)


@pytest.mark.parametrize("gemm_select", ["cublas", "zi", "auto"])
def test_fused_kernels_match_torch_path(gemm_select):
    """libzinf LayerNorm / bias-grad / GELU-bwd / softmax-CE path vs the torch-op path,
    with every linear on cuBLAS, every linear on zi_gemm (bias / GELU / residual / GELU'
    epilogues), or the per-site timed choice."""
    a = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, fused=True, gemm_select=gemm_select)
    b = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, fused=False)
    assert a.fused and not b.fused and set(a.gsel) == set(eg._GEMM_SITES)
    if gemm_select != "auto":
        assert set(a.gsel.values()) == {gemm_select}
    a.capture_grads = b.capture_grads = True
    bs = batches_for(SMALL, 2)
    la, lb = a.step(bs).item(), b.step(bs).item()
    assert abs(la - lb) <= 2e-3 * abs(lb)
    for key in a.grad_shards:
        for r in range(2):
            assert rel(a.grad_shards[key][r].cpu().numpy(), b.grad_shards[key][r].cpu().numpy()) < 3e-2, key


def test_loss_decreases_and_world_sizes_agree():
    c = SMALL
    out = {}
    for world in (1, 2):
        eng = eg.GPTZeroEngine(c, LocalComm(world), lr=3e-3)
        # same global data: rank r of world 2 == half of the world-1 batch is not
        # needed here; compare loss trends only
        losses = [eng.step(batches_for(c, world, 0)).item() for _ in range(8)]
        assert losses[-1] < 0.8 * losses[0], losses
        out[world] = losses
    assert np.isfinite(out[1]).all() and np.isfinite(out[2]).all()


@pytest.mark.parametrize("params_host,slots", [(False, 3), (False, 12), (False, 10_000),
                                               (True, 12)])
def test_offload_matches_hbm(params_host, slots):
    """Optimizer states (and optionally bf16 params) in pinned host DRAM, streamed in
    small chunks through the staging ring (prefetched across the step boundary, write-back
    deferred into the next forward): same result as all-in-HBM. slots=10_000 clamps the
    ring to the step's chunk count, the edge of the slot-reuse ordering argument."""
    from paper_2104_07857_b200.gpt import Placement
    from paper_2104_07857_b200.store import TierKind
    a = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3)
    pl = Placement(params=TierKind.HOST if params_host else TierKind.DEVICE, optim=TierKind.HOST)
    b = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, placement=pl, offload_chunk=10_007,
                         offload_slots=slots)
    assert len(b.stage) <= len(b._ochunks)
    assert not b.p32.is_cuda and b.p32.is_pinned()
    for step in range(3):
        bs = batches_for(SMALL, 2, step)
        la, lb = a.step(bs).item(), b.step(bs).item()
        assert la == lb, (step, la, lb)
    torch.cuda.synchronize()
    for key in a.by_key:
        for r in range(2):
            sa, sb = a.shard(key, r), b.shard(key, r)
            for n in ("p32", "m", "v"):
                torch.testing.assert_close(sa[n].cpu(), sb[n].cpu(), rtol=0, atol=0)
            assert torch.equal(sa["p16"].cpu(), sb["p16"].cpu())
    assert b.offload_bytes > 0


@pytest.mark.parametrize("direct", [False, True])
def test_nvme_optimizer_states_match_hbm(tmp_path, direct):
    """Optimizer states in NVMe .shard files streamed nc -> cg -> RS+Adam -> D2H -> nc in
    small chunks (through the page cache, or the native O_DIRECT engine): the same
    training result as keeping them in HBM."""
    from paper_2104_07857_b200.gpt import Placement
    from paper_2104_07857_b200.store import SHARD_MAGIC, TierKind
    a = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3)
    b = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, nvme_root=str(tmp_path),
                         placement=Placement(TierKind.DEVICE, TierKind.NVME), nvme_direct=direct)
    b.streamer.chunk = 30_000   # several chunks per bucket
    for step in range(3):
        bs = batches_for(SMALL, 2, step)
        la, lb = a.step(bs).item(), b.step_graphed(bs).item()
        assert la == lb, (step, la, lb)
    for key in a.by_key:
        for r in range(2):
            sa, sb = a.shard(key, r), b.shard(key, r)
            for n in ("p32", "m", "v"):
                np.testing.assert_allclose(sa[n].cpu().numpy(), sb[n].numpy(), rtol=0, atol=0)
    files = sorted(p.name for p in tmp_path.iterdir())
    assert "h0.p32%2Frank1.shard" in files
    assert (tmp_path / "h0.m%2Frank0.shard").read_bytes()[:4] == SHARD_MAGIC
    assert b.streamer.bytes > 0
    b.close()


def test_traced_timeline():
    """Real CUDA-event Timeline: gathers overlap compute on their own lane."""
    from paper_2104_07857_b200.gpt import Placement
    from paper_2104_07857_b200.store import TierKind
    eng = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, trace=True,
                           placement=Placement(TierKind.DEVICE, TierKind.HOST), offload_chunk=5000)
    eng.step(batches_for(SMALL, 2))
    tl = eng.timeline()
    stages = {e[1] for e in tl.events}
    assert {"compute", "gg", "cg", "grad_offload"} <= stages
    for op, st, lane, s, e in tl.events:
        assert e >= s >= 0
    assert 0.0 <= tl.hidden_fraction() <= 1.0
    assert tl.to_csv().count("\n") == len(tl.events) + 1
    # calibration: measured per-op costs replayed through the simulator
    fwd, bwd = eng.timeline("forward"), eng.timeline("backward")
    assert len(fwd.events) + len(bwd.events) == len(tl.events)
    assert {e[0] for e in fwd.events if e[1] == "compute"} == {b.op for b in eng.buckets[:-1]}
    from paper_2104_07857_b200.schedule import verify_timeline
    for duplex in (False, True):
        sim = eng.simulated_step(duplex)
        verify_timeline(sim["forward"])
        verify_timeline(sim["backward"])
        assert 0 < sim["predicted_s"] <= sim["serial_s"] + 1e-12
        assert sim["measured_s"] == tl.total_s


def test_copy_engine_gather_same_result():
    a = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3)
    b = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, copy_engine_gather=True, prefetch=False)
    bs = batches_for(SMALL, 2)
    la, lb = a.step(bs).item(), b.step(bs).item()
    assert la == lb                         # deterministic step: bitwise
    for key in a.by_key:
        torch.testing.assert_close(a.shard(key, 1)["p32"], b.shard(key, 1)["p32"],
                                   rtol=0, atol=0)


@pytest.mark.parametrize("params_host", [False, True])
def test_offload_graphed_matches_eager(params_host):
    """The optimizer-offload step captured into a CUDA graph (H2D / rs_adam / D2H chunk
    pipeline as graph nodes) trains exactly like the eager step."""
    from paper_2104_07857_b200.gpt import Placement
    from paper_2104_07857_b200.store import TierKind
    pl = Placement(params=TierKind.HOST if params_host else TierKind.DEVICE, optim=TierKind.HOST)
    a = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, placement=pl, offload_chunk=10_007,
                         gemm_select="zi")
    b = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, placement=pl, offload_chunk=10_007,
                         gemm_select="zi")
    for step in range(3):
        bs = batches_for(SMALL, 2, step)
        la, lb = a.step(bs).item(), b.step_graphed(bs).item()
        assert la == lb, (step, la, lb)
    for key in a.by_key:
        for r in range(2):
            sa, sb = a.shard(key, r), b.shard(key, r)
            torch.testing.assert_close(sa["p32"].cpu(), sb["p32"].cpu(), rtol=0, atol=0)


@pytest.mark.parametrize("K,params_host,graph", [(1, False, False), (2, True, False),
                                                 (99, True, False), (2, True, True)])
def test_param_reuse_cache_matches(K, params_host, graph):
    """param_cache=K keeps the forward's last K blocks gathered for the backward: same
    training as K=0 (K=99 clamps to every block but the first), and K fewer parameter
    fetches per step (host bytes with params on the host)."""
    from paper_2104_07857_b200.gpt import Placement
    from paper_2104_07857_b200.store import TierKind
    pl = Placement(params=TierKind.HOST if params_host else TierKind.DEVICE,
                   optim=TierKind.HOST if params_host else TierKind.DEVICE)
    cfg = eg.GPTConfig(nl=5, hd=128, heads=2, seq=128, vocab=256, batch=2)
    kw = dict(lr=1e-3, placement=pl, offload_chunk=10_007, gemm_select="zi")
    a = eg.GPTZeroEngine(cfg, LocalComm(2), **kw)
    b = eg.GPTZeroEngine(cfg, LocalComm(2), param_cache=K, **kw)
    assert b.K == min(K, cfg.nl - 1) and len(b.slots) == 2 + b.K
    for step in range(3):
        bs = batches_for(cfg, 2, step)
        la = a.step(bs).item()
        lb = (b.step_graphed if graph else b.step)(bs).item()
        assert la == lb, (step, la, lb)
    torch.cuda.synchronize()
    for key in a.by_key:
        for r in range(2):
            torch.testing.assert_close(a.shard(key, r)["p32"].cpu(), b.shard(key, r)["p32"].cpu(),
                                       rtol=0, atol=0)
    if params_host and not graph:
        blk = a.buckets[1].shard * 2 * 2                 # one block's bf16 shards, 2 ranks
        assert a.fetch_bytes - b.fetch_bytes == 3 * b.K * blk


def test_step_bitwise_reproducible():
    """The whole partitioned step is deterministic (fixed-order attention backward and
    embedding gradient, rank-order RS): two engines on the same data agree bit for bit."""
    runs = []
    for _ in range(2):
        e = eg.GPTZeroEngine(eg.TINY, LocalComm(2), lr=1e-3)
        losses = [e.step(batches_for(eg.TINY, 2, s)).item() for s in range(3)]
        runs.append((losses, {k: [e.shard(k, r)["p32"].cpu() for r in range(2)] for k in e.by_key}))
        del e
    assert runs[0][0] == runs[1][0]
    for k in runs[0][1]:
        for r in range(2):
            assert torch.equal(runs[0][1][k][r], runs[1][1][k][r]), k


def test_deferred_folds_bitwise_equal(monkeypatch):
    """The block backward's folds as one zi_fold_sets launch (default) == one fold per
    producer (ZI_FOLD_DEFER=0): same losses and master shards bit for bit."""
    runs = []
    for defer in ("1", "0"):
        monkeypatch.setenv("ZI_FOLD_DEFER", defer)
        e = eg.GPTZeroEngine(eg.TINY, LocalComm(2), lr=1e-3)
        assert e.fold_defer == (defer == "1")
        losses = [e.step(batches_for(eg.TINY, 2, s)).item() for s in range(2)]
        runs.append((losses, {k: [e.shard(k, r)["p32"].cpu() for r in range(2)] for k in e.by_key}))
        del e
    assert runs[0][0] == runs[1][0]
    for k in runs[0][1]:
        for r in range(2):
            assert torch.equal(runs[0][1][k][r], runs[1][1][k][r]), k
