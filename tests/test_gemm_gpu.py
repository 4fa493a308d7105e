"""tcgen05 tile GEMM (zi_linear_fwd) against an fp32 torch reference.

Tolerance: the kernel accumulates in fp32 and rounds once to bf16, so the
result must lie within 1 bf16 ulp (2^-7 relative) of the fp32 reference
plus a small absolute term for accumulation-order differences.
"""

import pytest
import torch

from paper_2104_07857_b200 import kernels

pytestmark = pytest.mark.gpu


def ref(x, w, b):
    y = x.float() @ w.float().t()
    if b is not None:
        y = y + b.float()
    return y


def check(y, yr, K):
    # one bf16 ulp (2^-7 relative): RNE is half an ulp, and fp32 accumulation-order
    # differences vs the reference can move a value across a rounding boundary
    # plus K * 2^-20 absolute: fp32 sums of K O(1) products in a different order
    # differ by ~K * eps32 where the result cancels to near zero
    err = (y.float() - yr).abs()
    tol = yr.abs() * 2 ** -7 + K * 2 ** -20
    bad = (err > tol).sum().item()
    assert bad == 0, f"{bad} elements out of tolerance; max err {err.max().item()}"


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 1024), (300, 520, 200),
                                   (1, 8, 8), (1000, 4104, 4096), (2048, 2048, 16384)])
@pytest.mark.parametrize("bias", [False, True])
def test_linear_fwd(M, N, K, bias):
    torch.manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * K ** -0.5
    b = torch.randn(N, device="cuda", dtype=torch.bfloat16) if bias else None
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    kernels.linear_fwd(x, w, b, y)
    torch.cuda.synchronize()
    check(y, ref(x, w, b), K)


@pytest.mark.parametrize("T,din,dout", [(256, 512, 1024), (1000, 320, 200), (8192, 2048, 6144)])
@pytest.mark.parametrize("f32", [False, True])
def test_backward_gemms(T, din, dout, f32):
    """dx = dy W (B N-major) and dW = dy^T x (A and B MN-major) on tcgen05."""
    torch.manual_seed(T + din)
    x = torch.randn(T, din, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(dout, din, device="cuda", dtype=torch.bfloat16) * din ** -0.5
    dy = torch.randn(T, dout, device="cuda", dtype=torch.bfloat16)
    odt = torch.float32 if f32 else torch.bfloat16
    dx = torch.empty(T, din, device="cuda", dtype=odt)
    kernels.gemm(dy, w.t(), dx)
    dW = torch.empty(dout, din, device="cuda", dtype=odt)
    kernels.gemm(dy.t(), x.t(), dW)
    torch.cuda.synchronize()
    check(dx, dy.float() @ w.float(), dout)
    check(dW, dy.float().t() @ x.float(), T)


def test_accumulate_fp32():
    """dx += g_t W_t over tiles (backward_tiled's running sum) in fp32."""
    torch.manual_seed(0)
    T, din, dout = 512, 768, 1024
    g = torch.randn(T, dout, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(dout, din, device="cuda", dtype=torch.bfloat16) * din ** -0.5
    acc = torch.zeros(T, din, device="cuda", dtype=torch.float32)
    for s in range(0, dout, 256):
        kernels.gemm(g[:, s:s + 256], w[s:s + 256].t(), acc, accumulate=True)
    torch.cuda.synchronize()
    ref = g.float() @ w.float()
    assert ((acc - ref).abs() <= 1e-3 * (1 + ref.abs())).all()


def test_linear_fwd_strided_views():
    """Tiles of a larger weight / output (ld > row length), as forward_tiled uses them."""
    M, K, Nfull, T = 256, 512, 1024, 4
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(Nfull, K, device="cuda", dtype=torch.bfloat16) * K ** -0.5
    y = torch.zeros(M, Nfull, device="cuda", dtype=torch.bfloat16)
    R = Nfull // T
    for t in range(T):
        kernels.linear_fwd(x, w[t * R:(t + 1) * R], None, y[:, t * R:(t + 1) * R])
    torch.cuda.synchronize()
    check(y, ref(x, w, None), K)
