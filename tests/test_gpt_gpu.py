"""The partitioned GPT step on the GPU against the CPU oracle (oracle/gpt.py).

Layout and init are bit-exact; gradients / loss within stated tolerances:
fp32 compute (half params widened, as the SPEC harness computes)
within 1e-5 on the loss and 1e-2 relative L2 on gradient shards (bucket
grads are rounded to half before the reduce-scatter, so summation-order
differences can flip single half ulps); bf16 compute within 2e-2 on the
loss and 6e-2 on gradients (SURVEY.md §8c tolerance proposal).
"""

import numpy as np
import pytest
import torch

from oracle import gpt as og
from oracle import numerics as nx
from paper_2104_07857_b200 import gpt as eg
from paper_2104_07857_b200.comm import LocalComm

pytestmark = pytest.mark.gpu

SMALL = eg.GPTConfig(nl=2, hd=128, heads=2, seq=64, vocab=256, batch=2)


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


@pytest.mark.parametrize("world", [1, 2])
def test_step_fp32_compute_matches_oracle(world):
    torch.backends.cuda.matmul.allow_tf32 = False
    eng = eg.GPTZeroEngine(SMALL, LocalComm(world), half_dtype=torch.float16,
                           compute_dtype=torch.float32, lr=1e-3)
    eng.capture_grads = True
    st = og.init_partitioned(ocfg(SMALL), world, half_kind=nx.HALF_FP16)
    for step in range(2):
        bs = batches_for(SMALL, world, step)
        loss = eng.step(bs).item()
        oloss, gsh = og.train_step(st, [(t.cpu().numpy(), y.cpu().numpy()) for t, y in bs], lr=1e-3)
        assert abs(loss - oloss) <= 1e-5 * abs(oloss), (step, loss, oloss)
        for key in gsh:
            for r in range(world):
                g = eng.grad_shards[key][r].cpu().numpy()
                assert rel(g, gsh[key][r]) < 1e-2, (step, key, r, rel(g, gsh[key][r]))
        for key in st.p32:
            for r in range(world):
                p = eng.shard(key, r)["p32"].cpu().numpy()
                assert np.abs(p - st.p32[key][r]).max() < 3e-3, key


def test_step_bf16_matches_oracle():
    world = 2
    eng = eg.GPTZeroEngine(SMALL, LocalComm(world), lr=1e-3)
    eng.capture_grads = True
    st = og.init_partitioned(ocfg(SMALL), world, half_kind=nx.HALF_BF16)
    bs = batches_for(SMALL, world)
    loss = eng.step(bs).item()
    oloss, gsh = og.train_step(st, [(t.cpu().numpy(), y.cpu().numpy()) for t, y in bs], lr=1e-3)
    assert abs(loss - oloss) <= 2e-2 * abs(oloss)
    for key in gsh:
        for r in range(world):
            assert rel(eng.grad_shards[key][r].cpu().numpy(), gsh[key][r]) < 6e-2, key


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
    np.testing.assert_allclose(la, lb, rtol=2e-5)
    assert int(a.adam.step.item()) == int(b.adam.step.item()) == 5
    for key in a.by_key:
        torch.testing.assert_close(a.shard(key, 0)["p32"], b.shard(key, 0)["p32"], rtol=0, atol=5e-5)


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
        assert abs(la - lb) <= 1e-5 * abs(la), (step, la, lb)
    for key in a.by_key:
        torch.testing.assert_close(a.shard(key, 1)["p32"], b.shard(key, 1)["p32"], rtol=0, atol=5e-5)
    if mode == "host":
        assert b.ckpt_bytes > 0
        stages = {e[1] for e in b.timeline().events}
        assert {"cg", "grad_offload", "compute"} <= stages


@pytest.mark.parametrize("hd,heads", [(4096, 32), (8192, 64)])
def test_10b_70b_layer_shapes(hd, heads):
    """One block at the 10B / 70B widths (BASELINE configs 3 and 5): the libzinf path
    agrees with the torch-op path."""
    c = eg.GPTConfig(nl=1, hd=hd, heads=heads, seq=64, vocab=512, batch=1)
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
        assert abs(la - lb) <= 1e-5 * abs(la), (step, la, lb)
    torch.cuda.synchronize()
    for key in a.by_key:
        for r in range(2):
            sa, sb = a.shard(key, r), b.shard(key, r)
            for n in ("p32", "m", "v"):
                torch.testing.assert_close(sa[n].cpu(), sb[n].cpu(), rtol=0, atol=5e-5)
            assert (sa["p16"].cpu().float() - sb["p16"].cpu().float()).abs().max() < 1e-2
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
        assert abs(la - lb) <= 1e-5 * abs(la), (step, la, lb)
    for key in a.by_key:
        for r in range(2):
            sa, sb = a.shard(key, r), b.shard(key, r)
            for n in ("p32", "m", "v"):
                np.testing.assert_allclose(sa[n].cpu().numpy(), sb[n].numpy(), rtol=0, atol=5e-5)
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
    assert abs(la - lb) <= 1e-6 * abs(la)   # atomics in attention/embedding bwd
    for key in a.by_key:
        torch.testing.assert_close(a.shard(key, 1)["p32"], b.shard(key, 1)["p32"],
                                   rtol=0, atol=2e-5)


@pytest.mark.parametrize("params_host", [False, True])
def test_offload_graphed_matches_eager(params_host):
    """The optimizer-offload step captured into a CUDA graph (H2D / rs_adam / D2H chunk
    pipeline as graph nodes) trains exactly like the eager step."""
    from paper_2104_07857_b200.gpt import Placement
    from paper_2104_07857_b200.store import TierKind
    pl = Placement(params=TierKind.HOST if params_host else TierKind.DEVICE, optim=TierKind.HOST)
    a = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, placement=pl, offload_chunk=10_007,
                         gemm_select="cublas")
    b = eg.GPTZeroEngine(SMALL, LocalComm(2), lr=1e-3, placement=pl, offload_chunk=10_007,
                         gemm_select="cublas")
    for step in range(3):
        bs = batches_for(SMALL, 2, step)
        la, lb = a.step(bs).item(), b.step_graphed(bs).item()
        assert abs(la - lb) <= 1e-5 * abs(la), (step, la, lb)
    for key in a.by_key:
        for r in range(2):
            sa, sb = a.shard(key, r), b.shard(key, r)
            torch.testing.assert_close(sa["p32"].cpu(), sb["p32"].cpu(), rtol=0, atol=5e-5)


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
    cfg = eg.GPTConfig(nl=5, hd=128, heads=2, seq=64, vocab=256, batch=2)
    kw = dict(lr=1e-3, placement=pl, offload_chunk=10_007, gemm_select="cublas")
    a = eg.GPTZeroEngine(cfg, LocalComm(2), **kw)
    b = eg.GPTZeroEngine(cfg, LocalComm(2), param_cache=K, **kw)
    assert b.K == min(K, cfg.nl - 1) and len(b.slots) == 2 + b.K
    for step in range(3):
        bs = batches_for(cfg, 2, step)
        la = a.step(bs).item()
        lb = (b.step_graphed if graph else b.step)(bs).item()
        assert abs(la - lb) <= 1e-5 * abs(la), (step, la, lb)
    torch.cuda.synchronize()
    for key in a.by_key:
        for r in range(2):
            torch.testing.assert_close(a.shard(key, r)["p32"].cpu(), b.shard(key, r)["p32"].cpu(),
                                       rtol=0, atol=5e-5)
    if params_host and not graph:
        blk = a.buckets[1].shard * 2 * 2                 # one block's bf16 shards, 2 ranks
        assert a.fetch_bytes - b.fetch_bytes == 3 * b.K * blk
