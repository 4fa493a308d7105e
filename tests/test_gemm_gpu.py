"""tcgen05 tile GEMM (zi_linear_fwd) against an fp32 torch reference.

Tolerance: the kernel accumulates in fp32 and rounds once to bf16, so the
result must lie within 1 bf16 ulp (2^-8 relative) of the fp32 reference
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
    err = (y.float() - yr).abs()
    tol = yr.abs() * 2 ** -8 + 1e-3 * (K ** 0.5) * 2 ** -8
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
