"""The CPU oracle against the SPEC's known answers and acceptance criteria (CPU only).

Pins: SPEC.md:470-471 (ceil split / pad), 646 (tile rows), 765 (Adam hand
step), 764 + AC-10 (chunk invariance), 505-506 (partition/allgather and
RS properties), AC-8 (tiling equivalence), AC-9 (placement / world
invariance + loss halving), AC-12 (finite-difference gradients).
"""

import json
import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import gpt as og
from oracle import harness as oh
from oracle import numerics as nx
from oracle.adam import AdamConsts, adam_update, chunked_adam_step
from oracle.partition import allgather, partition, reduce_scatter, shard_len
from oracle.schedule import plan_prefetch
from oracle.tiling import backward_tiled, forward_tiled, peak_tile_bytes, tile_rows

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


def test_spec_examples(gold):
    for n, w, L in gold["shard_len"]:
        assert shard_len(n, w) == L
    assert shard_len(10, 4) == 3
    assert int((partition(np.arange(1, 11, dtype=np.float32), 4)[3] == 0).sum()) == 2
    assert [e - s for s, e in tile_rows(10, 4)] == [3, 3, 3, 1] == gold["tile_rows_10_4"]
    assert partition(np.arange(5.0), 1)[0].tolist() == list(np.arange(5.0))


def test_adam_hand_step(gold):
    c = AdamConsts.make(0.1, 0.9, 0.999, 1e-8, 1)
    P, M, V = adam_update(np.ones(1, np.float32), np.zeros(1, np.float32),
                          np.zeros(1, np.float32), np.ones(1, np.float32), c)
    assert abs(M[0] - 0.1) < 1e-7 and abs(V[0] - 0.001) < 1e-9 and abs(P[0] - 0.9) < 1e-6
    assert int(P.view(np.uint32)[0]) == gold["adam_hand"]["p_bits"]


def test_numerics_golden(gold):
    got = nx.uniform_init(7, 65, 0, 16, 1 / 2048 ** 0.5).view(np.uint32).tolist()
    assert got == gold["uniform_init_seed7_stream65_first16"]
    for x, b in gold["bf16_rne"].items():
        assert int(nx.f32_to_bf16_bits(np.array([float(x)], np.float32))[0]) == b
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32)
    # bf16 RNE agrees with float64 nearest-even reference rounding
    b = nx.bf16_bits_to_f32(nx.f32_to_bf16_bits(x))
    assert np.all(np.abs(b - x) <= np.abs(x) * 2 ** -8)
    # shard-local generation == slicing the full stream
    full = nx.uniform_init(3, 9, 0, 1000, 0.5)
    assert np.array_equal(nx.uniform_init(3, 9, 400, 250, 0.5), full[400:650])


@settings(max_examples=200, deadline=None)
@given(n=st.integers(1, 10_000), world=st.integers(1, 17),
       dt=st.sampled_from([np.float16, np.float32, np.float64]))
def test_partition_allgather_identity(n, world, dt):
    """partition o allgather = identity for lengths 1..1e4, world 1..17."""
    x = np.random.default_rng(n).standard_normal(n).astype(dt)
    shards = partition(x, world)
    assert len(shards) == world and all(s.size == shard_len(n, world) for s in shards)
    assert np.array_equal(allgather(shards, n), x)
    pad = world * shard_len(n, world) - n
    assert not np.concatenate(shards)[n:].any() and np.concatenate(shards)[n:].size == pad


@settings(max_examples=100, deadline=None)
@given(n=st.integers(1, 3000), world=st.integers(1, 9), dt=st.sampled_from([np.float32, np.float64]))
def test_rs_then_ag_is_sequential_sum(n, world, dt):
    """RS o AG equals the sequential elementwise sum, bit-exact."""
    rng = np.random.default_rng(n * 31 + world)
    cs = [rng.standard_normal(n).astype(dt) for _ in range(world)]
    s = cs[0].copy()
    for c in cs[1:]:
        s = s + c
    assert np.array_equal(allgather(reduce_scatter(cs, world), n), s)


@pytest.mark.parametrize("chunk", [1, 3, 64, 10_000])
def test_chunk_invariance(chunk):
    n = 1000
    rng = np.random.default_rng(5)
    p, m, g = (rng.standard_normal(n).astype(np.float32) for _ in range(3))
    v = np.abs(rng.standard_normal(n)).astype(np.float32)
    c = AdamConsts.make(1e-3, 0.9, 0.999, 1e-8, 7)
    ref = chunked_adam_step(p, m, v, g, c, n, nx.HALF_FP16)
    got = chunked_adam_step(p, m, v, g, c, chunk, nx.HALF_FP16)
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("T", [1, 2, 3, 4, 7, 16])
@pytest.mark.parametrize("dt,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
def test_tiling_equivalence(T, dt, tol):
    """AC-8 on sizes up to 128x512."""
    rng = np.random.default_rng(T)
    W = rng.standard_normal((128, 512)).astype(dt)
    b = rng.standard_normal(128).astype(dt)
    x = rng.standard_normal((16, 512)).astype(dt)
    gy = rng.standard_normal((16, 128)).astype(dt)
    y = forward_tiled(W, b, x, T)
    yd = x @ W.T + b
    assert np.abs(y - yd).max() / np.abs(yd).max() < tol
    dW, db, dx = backward_tiled(W, x, gy, T)
    for a, e in ((dW, gy.T @ x), (db, gy.sum(0)), (dx, gy @ W)):
        assert np.abs(a - e).max() / np.abs(e).max() < tol
    assert peak_tile_bytes(128, 512, T, 8) <= -(-(128 * 512 * 8) // T) + 512 * 8
    assert np.array_equal(forward_tiled(W, b, np.zeros_like(x), T), np.broadcast_to(b, (16, 128)))


def toy_spec(tied=False, tiled=False):
    L = oh.LayerSpec
    if not tied and not tiled:
        return oh.ModelSpec([L("linear", 8, 16, "relu"), L("linear", 16, 16, "relu"),
                             L("linear", 16, 4)], seed=7)
    return oh.ModelSpec([L("linear", 8, 16, "relu"),
                         L("tiled_linear", 16, 16, "gelu-approx", tiles=4),
                         L("linear", 16, 16, "relu"), L("linear", 16, 16, "relu"),
                         L("linear", 16, 4)], tied_pairs=[(2, 3)], seed=7)


@pytest.mark.parametrize("variant", [dict(), dict(tied=True, tiled=True)])
def test_ac9_world_invariance_and_convergence(variant):
    spec = toy_spec(**variant)
    d1, l1 = oh.run_training(spec, 1, 50)
    d4, l4 = oh.run_training(spec, 4, 50, chunk_elems=3)
    assert d1 == d4 and l1 == l4
    assert l1[-1] < 0.5 * l1[0]


def test_ac12_gradient_check_toy():
    spec = oh.ModelSpec([oh.LayerSpec("linear", 8, 16, "gelu-approx"),
                         oh.LayerSpec("linear", 16, 4)], seed=3)
    bk = {k: v.astype(np.float64) for k, v in oh.init_buckets(spec).items()}
    x, t = oh.synthetic_batch(spec, 8)
    loss, g = oh.forward_backward(spec, bk, x, t, 32.0, np.float64)
    h = 1e-6
    for k in bk:
        for i in range(0, bk[k].size, 7):
            p = {kk: v.copy() for kk, v in bk.items()}
            m = {kk: v.copy() for kk, v in bk.items()}
            p[k][i] += h
            m[k][i] -= h
            fd = (oh.forward_backward(spec, p, x, t, 32.0, np.float64)[0] -
                  oh.forward_backward(spec, m, x, t, 32.0, np.float64)[0]) / (2 * h)
            assert abs(fd - g[k][i]) <= 1e-6 * max(1.0, abs(fd)) + 1e-9


def test_ac12_gradient_check_gpt():
    c = og.GPTConfig(nl=1, hd=16, heads=2, seq=8, vocab=32, batch=2)
    st_ = og.init_partitioned(c, 1)
    full = {k: v.astype(np.float64) for k, v in og.gathered(st_).items()}
    tok, tgt = og.synthetic_tokens(c, 7, 0)
    _, g = og.forward_backward(c, full, tok, tgt, dtype=np.float64)
    rng = np.random.default_rng(0)
    h = 1e-6
    for k in full:
        for i in rng.integers(0, full[k].size, 8):
            p = {kk: v.copy() for kk, v in full.items()}
            m = {kk: v.copy() for kk, v in full.items()}
            p[k][i] += h
            m[k][i] -= h
            fd = (og.forward_backward(c, p, tok, tgt, dtype=np.float64)[0] -
                  og.forward_backward(c, m, tok, tgt, dtype=np.float64)[0]) / (2 * h)
            assert abs(fd - g[k][i]) <= 1e-6 * max(1e-3, abs(fd)), (k, i, fd, g[k][i])


def test_plan_prefetch_examples():
    plan = plan_prefetch(5, (3, 2, 1))
    assert plan[1] == {"at": 0, "nc": [3], "cg": [2], "gg": [1]}
    assert plan[0]["nc"] == [0, 1, 2] and plan[0]["gg"] == [0]
    one = plan_prefetch(1, (3, 2, 1))
    assert one[0] == {"at": -1, "nc": [0], "cg": [0], "gg": [0]}
    with pytest.raises(ValueError):
        plan_prefetch(4, (1, 2, 1))
