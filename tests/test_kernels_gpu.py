"""Parity of the libzinf kernels against the CPU oracle (bit-exact), on the GPU.

Sizes include ragged tails (not multiples of 8), misaligned offsets, a
single element, and config-1 / config-2 shard sizes.
"""

import numpy as np
import pytest
import torch

from oracle import numerics as nx
from oracle.adam import AdamConsts, adam_update, chunked_adam_step, rs_adam
from oracle.partition import allgather as o_allgather
from oracle.partition import partition as o_partition
from oracle.partition import reduce_scatter as o_rs
from paper_2104_07857_b200 import _lib, kernels

pytestmark = pytest.mark.gpu

HALVES = [(torch.bfloat16, nx.HALF_BF16), (torch.float16, nx.HALF_FP16)]


def bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)


def f32(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def dev_half(bits16: np.ndarray, dtype) -> torch.Tensor:
    return torch.from_numpy(bits16.view(np.int16).copy()).view(dtype).cuda()


@pytest.mark.parametrize("n", [1, 7, 8, 1000, 4099, 1_661_696])
@pytest.mark.parametrize("half", HALVES)
def test_adam_bit_exact(n, half):
    dt, kind = half
    rng = np.random.default_rng(n)
    p = rng.uniform(-0.05, 0.05, n).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v = np.abs(rng.standard_normal(n) * 1e-6).astype(np.float32)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    for step in (1, 2, 1000):
        c = AdamConsts.make(1e-4, 0.9, 0.999, 1e-8, step)
        P, M, V = adam_update(p, m, v, g, c)
        tp, tm, tv, tg = (torch.from_numpy(a.copy()).cuda() for a in (p, m, v, g))
        th = torch.empty(n, dtype=dt, device="cuda")
        kernels.adam_step(tp, tm, tv, tg, th, _lib.adam_consts(1e-4, 0.9, 0.999, 1e-8, step))
        torch.cuda.synchronize()
        assert np.array_equal(f32(tp).view(np.uint32), P.view(np.uint32))
        assert np.array_equal(f32(tm).view(np.uint32), M.view(np.uint32))
        assert np.array_equal(f32(tv).view(np.uint32), V.view(np.uint32))
        assert np.array_equal(bits(th), nx.f32_to_half_bits(P, kind))


def test_adam_hand_step():
    """p=1, g=1, m=v=0, lr=0.1, betas (0.9, 0.999) -> m=0.1, v=0.001, p~0.9."""
    t = lambda x: torch.tensor([x], dtype=torch.float32, device="cuda")
    p, m, v, g = t(1.0), t(0.0), t(0.0), t(1.0)
    h = torch.empty(1, dtype=torch.float16, device="cuda")
    kernels.adam_step(p, m, v, g, h, _lib.adam_consts(0.1, 0.9, 0.999, 1e-8, 1))
    assert abs(m.item() - 0.1) < 1e-7 and abs(v.item() - 0.001) < 1e-9
    assert abs(p.item() - 0.9) < 1e-6
    assert h.item() == np.float16(p.item())


def test_adam_misaligned_views():
    n = 1003
    base = [torch.randn(n + 3, device="cuda") for _ in range(4)]
    p, m, v, g = (b[1:1 + n] for b in base)
    v.abs_()
    pn, mn, vn, gn = (f32(x) for x in (p, m, v, g))
    c = AdamConsts.make(1e-3, 0.9, 0.95, 1e-8, 3)
    P, M, V = adam_update(pn, mn, vn, gn, c)
    kernels.adam_step(p, m, v, g, None, _lib.adam_consts(1e-3, 0.9, 0.95, 1e-8, 3))
    assert np.array_equal(f32(p).view(np.uint32), P.view(np.uint32))


@pytest.mark.parametrize("chunk", [1, 3, 64, 10_000])
def test_chunk_invariance_kernel(chunk):
    """AC-10: chunked updates through the kernel equal the oracle for any chunk size."""
    n = 777
    rng = np.random.default_rng(3)
    p, g = rng.standard_normal(n).astype(np.float32), rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    c = AdamConsts.make(1e-2, 0.9, 0.999, 1e-8, 1)
    P, M, V, H = chunked_adam_step(p, m, v, g, c, n, nx.HALF_FP16)
    tp, tm, tv, tg = (torch.from_numpy(a.copy()).cuda() for a in (p, m, v, g))
    th = torch.empty(n, dtype=torch.float16, device="cuda")
    cc = _lib.adam_consts(1e-2, 0.9, 0.999, 1e-8, 1)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        kernels.adam_step(tp[s:e], tm[s:e], tv[s:e], tg[s:e], th[s:e], cc)
    assert np.array_equal(f32(tp).view(np.uint32), P.view(np.uint32))
    assert np.array_equal(bits(th), H)


@pytest.mark.parametrize("world,n", [(1, 10), (2, 1001), (4, 10), (8, 65_543), (3, 4096), (17, 999)])
@pytest.mark.parametrize("half", HALVES)
def test_reduce_scatter_cast_bit_exact(world, n, half):
    dt, kind = half
    rng = np.random.default_rng(world * 1000 + n)
    L = -(-n // world)
    contribs = [nx.f32_to_half_bits(rng.standard_normal(n).astype(np.float32), kind)
                for _ in range(world)]
    widened = [nx.half_bits_to_f32(c, kind) for c in contribs]
    exp = o_rs(widened, world, np.float32)
    scale = 1.0 / world
    dc = [dev_half(c, dt) for c in contribs]
    for r in range(world):
        out = torch.empty(L, dtype=torch.float32, device="cuda")
        kernels.reduce_scatter_cast(dc, r * L, L, n, scale, dt, out)
        want = exp[r] * np.float32(scale)
        assert np.array_equal(f32(out).view(np.uint32), want.view(np.uint32)), r


@pytest.mark.parametrize("dtype,npdt", [(torch.float32, np.float32), (torch.float64, np.float64)])
def test_reduce_scatter_full_precision(dtype, npdt):
    """RS is bit-exact in f32 and f64 given the fixed order."""
    from paper_2104_07857_b200.partition import reduce_scatter
    world, n = 5, 12_345
    rng = np.random.default_rng(9)
    cs = [rng.standard_normal(n).astype(npdt) for _ in range(world)]
    exp = o_rs(cs, world)
    got = reduce_scatter([torch.from_numpy(c).cuda() for c in cs], world)
    for r in range(world):
        assert np.array_equal(got[r].cpu().numpy(), exp[r])


@pytest.mark.parametrize("world,n", [(1, 9), (2, 1_661_696 * 2 - 3), (8, 100_007)])
@pytest.mark.parametrize("half", HALVES)
def test_rs_adam_bit_exact(world, n, half):
    dt, kind = half
    rng = np.random.default_rng(n)
    L = -(-n // world)
    contribs = [nx.f32_to_half_bits((rng.standard_normal(n) * 1e-2).astype(np.float32), kind)
                for _ in range(world)]
    dc = [dev_half(c, dt) for c in contribs]
    c = AdamConsts.make(3e-4, 0.9, 0.95, 1e-8, 5)
    cc = _lib.adam_consts(3e-4, 0.9, 0.95, 1e-8, 5)
    for r in range(world):
        p = rng.uniform(-0.1, 0.1, L).astype(np.float32)
        m = (rng.standard_normal(L) * 1e-3).astype(np.float32)
        v = np.abs(rng.standard_normal(L) * 1e-5).astype(np.float32)
        P, M, V, H, G = rs_adam(p, m, v, contribs, r, world, 1.0 / world, c, kind)
        tp, tm, tv = (torch.from_numpy(a.copy()).cuda() for a in (p, m, v))
        th = torch.empty(L, dtype=dt, device="cuda")
        tg = torch.empty(L, dtype=torch.float32, device="cuda")
        kernels.rs_adam(dc, r * L, L, n, 1.0 / world, tp, tm, tv, th, cc, g_out=tg)
        assert np.array_equal(f32(tg).view(np.uint32), G.view(np.uint32))
        assert np.array_equal(f32(tp).view(np.uint32), P.view(np.uint32))
        assert np.array_equal(f32(tm).view(np.uint32), M.view(np.uint32))
        assert np.array_equal(f32(tv).view(np.uint32), V.view(np.uint32))
        assert np.array_equal(bits(th), H)


@pytest.mark.parametrize("world,n", [(1, 1), (4, 10), (3, 1000), (8, 1 << 20), (7, 123_457)])
@pytest.mark.parametrize("ce", [False, True])
def test_allgather_bit_exact(world, n, ce):
    rng = np.random.default_rng(n)
    full = rng.integers(0, 65535, n, dtype=np.uint16)
    shards = o_partition(full, world)
    ds = [torch.from_numpy(s.view(np.int16).copy()).cuda() for s in shards]
    L = shards[0].size
    out = torch.full((L * world,), -1, dtype=torch.int16, device="cuda")
    kernels.allgather(ds, L, out, n, use_copy_engine=ce)
    got = out[:n].cpu().numpy().view(np.uint16)
    assert np.array_equal(got, o_allgather(shards, n))
    # bytes beyond full_len are untouched (truncation)
    assert (out[n:].cpu().numpy() == -1).all()


@pytest.mark.parametrize("n,start", [(1, 0), (1000, 17), (4099, 1 << 33)])
@pytest.mark.parametrize("half", HALVES)
def test_init_uniform_bit_exact(n, start, half):
    dt, kind = half
    seed, stream, bound = 7, 65, 1 / np.sqrt(2048)
    want = nx.uniform_init(seed, stream, start, n, bound)
    key = nx.rng_key(seed, stream)
    m = torch.empty(n, dtype=torch.float32, device="cuda")
    h = torch.empty(n, dtype=dt, device="cuda")
    kernels.init_uniform(m, h, key, start, float(nx.uniform_scale(bound)))
    assert np.array_equal(f32(m).view(np.uint32), want.view(np.uint32))
    assert np.array_equal(bits(h), nx.f32_to_half_bits(want, kind))
    assert np.abs(want).max() < bound


@pytest.mark.parametrize("half", HALVES)
def test_casts_bit_exact(half):
    dt, kind = half
    x = (np.random.default_rng(1).standard_normal(100_003) * 100).astype(np.float32)
    x[:4] = [0.0, -0.0, 65504.0, 1e-8]
    t = torch.from_numpy(x).cuda()
    h = torch.empty(x.size, dtype=dt, device="cuda")
    kernels.cast_f32_to_half(t, h)
    assert np.array_equal(bits(h), nx.f32_to_half_bits(x, kind))
    back = torch.empty(x.size, dtype=torch.float32, device="cuda")
    kernels.cast_half_to_f32(h, back)
    assert np.array_equal(f32(back), nx.half_bits_to_f32(bits(h), kind))


def test_bad_arguments_raise():
    t = torch.zeros(8, device="cuda")
    with pytest.raises(ValueError):
        kernels.reduce_scatter_cast([], 0, 8, 8, 1.0, torch.bfloat16, t)
    with pytest.raises(ValueError):
        _lib.call("zi_adam_step", None, None, None, None, None, 8, None, 0, None)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_matmul_fixed_order(dtype):
    """zi_matmul_fixed: equals a sequential fma chain per output (checked against an fp64
    reference within the fp32 / fp64 rounding bound), accepts transposed views, and is
    bit-identical across calls and operand placements."""
    torch.manual_seed(0)
    M, K, N = 37, 19, 23
    a = torch.randn(M, K, dtype=dtype, device="cuda")
    w = torch.randn(N, K, dtype=dtype, device="cuda")
    b = torch.randn(N, dtype=dtype, device="cuda")
    y = kernels.matmul_fixed(a, w.t(), bias=b)
    ref = a.double() @ w.double().t() + b.double()
    eps = torch.finfo(dtype).eps
    assert (y.double() - ref).abs().max().item() <= 4 * K * eps * ref.abs().max().item()
    # same bits through a differently laid-out copy of the operands
    wt = w.t().contiguous()                 # (K, N) row-major: the same B, other strides
    big = torch.zeros(M + 5, K + 3, dtype=dtype, device="cuda")
    big[5:, 3:] = a
    y2 = kernels.matmul_fixed(big[5:, 3:], wt, bias=b)
    assert torch.equal(y, y2)
    yc = kernels.matmul_fixed(a.t().contiguous().t(), w.t())   # column-major A view
    assert torch.equal(yc, kernels.matmul_fixed(a, w.t()))
    with pytest.raises(ValueError):
        kernels.matmul_fixed(a, w)
