"""Stream-K tcgen05 GEMM (zi_gemm_sk) against an fp32 torch reference.

Tolerances as tests/test_gemm_gpu.py: one bf16 ulp (2^-7 relative) of the fp32
reference plus K * 2^-20 absolute (fp32 accumulation-order differences); fp32 output:
2^-20 relative + K * 2^-22 absolute. Epilogues compose a bf16 rounding of the
accumulator with a bf16 operand as the kernel does (the reference rounds at the same
points). The split (stream-K) schedule must be bitwise repeatable.
"""

import pytest
import torch

from paper_2104_07857_b200 import kernels

pytestmark = pytest.mark.gpu
bf = torch.bfloat16


def gelu(z):
    return torch.nn.functional.gelu(z, approximate="tanh")


def gelu_grad(z):
    th = torch.tanh(0.7978845608028654 * (z + 0.044715 * z ** 3))
    return 0.5 * (1 + th) + 0.5 * z * (1 - th * th) * 0.7978845608028654 * (1 + 3 * 0.044715 * z * z)


def check(y, yr, K, rel=2 ** -7, name="", extra=None):
    err = (y.float() - yr).abs()
    tol = yr.abs() * rel + K * 2 ** -20
    if extra is not None:       # operand-scaled slack of the composed epilogues
        tol = tol + extra
    bad = (err > tol).sum().item()
    assert bad == 0, f"{name}: {bad} elements out of tolerance; max err {err.max().item()}"


def operands(kind, M, N, K, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if kind == "fwd":      # a (M, K) K-major, b (N, K) K-major
        a = torch.randn(M, K, device="cuda", generator=g).to(bf)
        b = (torch.randn(N, K, device="cuda", generator=g) * K ** -0.5).to(bf)
        return a, b
    if kind == "dx":       # b = W^T view: W (K, N) row-major -> b (N, K) N-major
        a = torch.randn(M, K, device="cuda", generator=g).to(bf)
        w = (torch.randn(K, N, device="cuda", generator=g) * K ** -0.5).to(bf)
        return a, w.t()
    # dW: a = dy^T (M, K) M-major, b = x^T (N, K) N-major
    dy = torch.randn(K, M, device="cuda", generator=g).to(bf)
    x = (torch.randn(K, N, device="cuda", generator=g) * K ** -0.5).to(bf)
    return dy.t(), x.t()


# (cluster tiles of 256 x 512 on 37 preferred clusters of 4; stream-K over the T mod 37
# tiles of the last partial wave)
SHAPES = [
    (256, 256, 64),        # one tile
    (300, 520, 200),       # ragged M / N / K
    (2048, 2048, 8192),    # 32 tiles < 37 clusters: whole tiles
    (8192, 2048, 2048),    # 128 tiles: 3 whole waves + 17 tiles cut across 2-3 clusters
    (1000, 4104, 1024),    # ragged
    (8192, 6144, 2048),    # qkv: 384 tiles, 14 cut
    (8192, 2048, 128),     # 17 cut tiles x 2 k-blocks over 37 clusters: empty ranges
    (4096, 4608, 64),      # one k-block: 33 tail tiles, whole, 4 clusters idle
]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("kind", ["fwd", "dx", "dw"])
@pytest.mark.parametrize("split", [True, False])
def test_plain(M, N, K, kind, split):
    if kind == "dw" and M % 8:
        pytest.skip("an M-major A needs M % 8 == 0 (16-byte TMA rows)")
    a, b = operands(kind, M, N, K, M + N + K)
    bias = None
    if kind == "fwd":
        bias = torch.randn(N, device="cuda").to(bf)
    y = torch.empty(M, N, device="cuda", dtype=bf)
    kernels.gemm_sk(a, b, y, bias=bias, split=split)
    yr = a.float() @ b.float().t()
    if bias is not None:
        yr = yr + bias.float()
    torch.cuda.synchronize()
    check(y, yr, K, name=f"{kind} {M}x{N}x{K}")


@pytest.mark.parametrize("M,N,K", [(2048, 2048, 8192), (50304 // 8, 2048, 1024), (304, 520, 200)])
def test_f32_out(M, N, K):
    a, b = operands("dw", M, N, K, 3)
    y = torch.empty(M, N, device="cuda", dtype=torch.float32)
    kernels.gemm_sk(a, b, y)
    yr = a.double() @ b.double().t()
    torch.cuda.synchronize()
    err = (y.double() - yr).abs()
    assert (err <= yr.abs() * 2 ** -20 + K * 2 ** -22).all(), err.max().item()


@pytest.mark.parametrize("M,N,K", [(8192, 8192, 2048), (300, 520, 200), (2048, 4096, 1024)])
def test_epilogues(M, N, K):
    a, b = operands("fwd", M, N, K, 11)
    bias = torch.randn(N, device="cuda").to(bf)
    acc = a.float() @ b.float().t()
    u = (acc + bias.float()).to(bf)
    # bias + GELU, both outputs
    y, y2 = torch.empty(M, N, device="cuda", dtype=bf), torch.empty(M, N, device="cuda", dtype=bf)
    kernels.gemm_sk(a, b, y, bias=bias, epi="gelu", out2=y2)
    torch.cuda.synchronize()
    check(y, acc + bias.float(), K, name="gelu.u")
    # the GELU output is computed from the kernel's own bf16 u
    # (tanh.approx: ~2^-10 absolute on tanh, so |u| * 2^-10 on gelu)
    check(y2, gelu(y.float()), K, rel=2 ** -7, name="gelu.a", extra=y.float().abs() * 2 ** -10)
    # bias + residual
    x = torch.randn(M, N, device="cuda").to(bf)
    yr = torch.empty(M, N, device="cuda", dtype=bf)
    kernels.gemm_sk(a, b, yr, bias=bias, epi="resid", x=x)
    torch.cuda.synchronize()
    # one bf16 ulp of u (its rounding may differ from the reference's) plus the final one
    check(yr, u.float() + x.float(), K, name="resid", extra=u.float().abs() * 2 ** -7)
    # GELU' of the pre-activation (dx of fc2 -> du of fc1); no bias
    yd = torch.empty(M, N, device="cuda", dtype=bf)
    kernels.gemm_sk(a, b, yd, epi="dgelu", x=x)
    torch.cuda.synchronize()
    ref = acc.to(bf).float() * gelu_grad(x.float())
    check(yd, ref, K, name="dgelu", extra=acc.abs() * (gelu_grad(x.float()).abs() * 2 ** -7 + 2 ** -9))
    # GELU'-saving forward: D = GELU'(u), D2 = GELU(u) of the kernel's own bf16 u (the same
    # GELU bits as the "gelu" epilogue); then the multiply-only backward epilogue
    gp, ga = torch.empty(M, N, device="cuda", dtype=bf), torch.empty(M, N, device="cuda", dtype=bf)
    kernels.gemm_sk(a, b, gp, bias=bias, epi="gelu_save", out2=ga)
    torch.cuda.synchronize()
    assert torch.equal(ga.view(torch.int16), y2.view(torch.int16))
    check(gp, gelu_grad(y.float()), K, rel=2 ** -7, name="gelu_save.d",
          extra=(y.float().abs() + 1) * 2 ** -9)
    ym = torch.empty(M, N, device="cuda", dtype=bf)
    kernels.gemm_sk(a, b, ym, epi="mul", x=gp)
    torch.cuda.synchronize()
    check(ym, acc.to(bf).float() * gp.float(), K, name="mul", extra=acc.abs() * gp.float().abs() * 2 ** -7)


@pytest.mark.parametrize("M,N,K,kind", [(8192, 2048, 2048, "fwd"), (2048, 2048, 8192, "dw"),
                                        (1000, 4104, 1024, "dx")])
def test_split_is_deterministic(M, N, K, kind):
    """The stream-K partial sums are folded in a fixed order: repeated launches are
    bitwise identical (and the flags reset: launch k+1 does not see launch k's)."""
    a, b = operands(kind, M, N, K, 5)
    y0 = torch.empty(M, N, device="cuda", dtype=bf)
    kernels.gemm_sk(a, b, y0)
    for _ in range(5):
        y = torch.empty(M, N, device="cuda", dtype=bf)
        kernels.gemm_sk(a, b, y)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), y0.view(torch.int16))


def test_workspace_per_stream_and_graph():
    """A captured stream-K launch replays bitwise equal to the eager one."""
    a, b = operands("fwd", 8192, 2048, 2048, 9)
    y0 = torch.empty(8192, 2048, device="cuda", dtype=bf)
    kernels.gemm_sk(a, b, y0)
    y = torch.empty_like(y0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        kernels.gemm_sk(a, b, y)          # warm: the side stream's workspace
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        kernels.gemm_sk(a, b, y)
    for _ in range(3):
        y.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), y0.view(torch.int16))


def test_rejects_bad_arguments():
    a, b = operands("fwd", 256, 256, 64, 1)
    y = torch.empty(256, 256, device="cuda", dtype=torch.float32)
    with pytest.raises(ValueError):
        kernels.gemm_sk(a, b, y, epi="gelu", out2=y)
    with pytest.raises(ValueError):
        kernels.gemm_sk(a, b, y, bias=torch.zeros(256, device="cuda", dtype=bf))


@pytest.mark.parametrize("M,N,K,epi", [(8192, 8192, 2048, "dgelu"), (300, 520, 200, "dgelu"),
                                       (1000, 2056, 1024, "plain"), (8192, 2048, 2048, "plain")])
@pytest.mark.parametrize("split", [True, False])
def test_colsum_side_output(M, N, K, epi, split):
    """32-row block column sums of the stored bf16 output, folded in block order: the
    bias gradient of the fc1 layer from the fc2 input-gradient GEMM. Checked against
    the fp32 sum of the kernel's own bf16 output (exact up to fp32 summation order),
    bitwise repeatable; rows past M (bias-only epilogue values) never count."""
    a, b = operands("dx", M, N, K, 21)
    x = torch.randn(M, N, device="cuda").to(bf)
    bias = torch.randn(N, device="cuda").to(bf) if epi == "plain" else None
    y = torch.empty(M, N, device="cuda", dtype=bf)
    P = -(-M // 32)
    part = torch.full((P * N,), float("nan"), device="cuda")
    kernels.gemm_sk(a, b, y, bias=bias, epi=epi, x=x if epi == "dgelu" else None,
                    colsum=part, split=split)
    out = torch.empty(N, device="cuda")
    kernels.colsum_fold(part, P, N, out)
    ob = torch.empty(N, device="cuda", dtype=bf)
    kernels.colsum_fold(part, P, N, ob)
    torch.cuda.synchronize()
    ref = y.double().sum(0)
    assert torch.isfinite(out).all()
    torch.testing.assert_close(out.double(), ref, rtol=1e-5, atol=1e-5 * M ** 0.5)
    assert torch.equal(ob, out.to(bf))
    blk = y[:32 * (M // 32)].float().view(M // 32, 32, N).sum(1)
    torch.testing.assert_close(part.view(P, N)[:M // 32], blk, rtol=1e-5, atol=1e-5)
    part2 = torch.empty_like(part)
    kernels.gemm_sk(a, b, torch.empty_like(y), bias=bias, epi=epi,
                    x=x if epi == "dgelu" else None, colsum=part2, split=split)
    torch.cuda.synchronize()
    assert torch.equal(part, part2)


@pytest.mark.parametrize("B,S,H,D", [(8, 1024, 16, 128), (2, 256, 4, 64), (1, 128, 3, 128)])
def test_delta_side_output(B, S, H, D):
    """proj.dx epilogue: dO = dx2 Wp^T and delta[b, h, s] = sum over the head's D
    columns of bf16(dO) * O — the attention backward's rowsum(dO o O)."""
    M, N, K = B * S, H * D, H * D
    a, b = operands("dx", M, N, K, 5)
    o = torch.randn(M, N, device="cuda").to(bf)
    y = torch.empty(M, N, device="cuda", dtype=bf)
    delta = torch.full((B * H * S,), float("nan"), device="cuda")
    kernels.gemm_sk(a, b, y, x=o, delta=delta, delta_shape=(S, H, D))
    torch.cuda.synchronize()
    check(y, a.float() @ b.float().t(), K, name="dO")
    ref = (y.float() * o.float()).view(B, S, H, D).sum(-1).permute(0, 2, 1).reshape(-1)
    torch.testing.assert_close(delta, ref, rtol=1e-5, atol=1e-4)
    d2 = torch.empty_like(delta)
    kernels.gemm_sk(a, b, torch.empty_like(y), x=o, delta=d2, delta_shape=(S, H, D))
    torch.cuda.synchronize()
    assert torch.equal(delta, d2)
