"""Wide-tile GEMM with each fused epilogue vs cuBLAS on the GPT shapes (TFLOP/s)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels  # noqa: E402


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


for M, N, K in [(8192, 8192, 2048), (8192, 6144, 2048), (8192, 2048, 8192), (8192, 8192, 8192)]:
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = 2 * M * N * K / 1e9
    y2 = torch.empty_like(y)
    r = {"plain": f / t(lambda: kernels.gemm_ex(x, w, y)),
         "gelu": f / t(lambda: kernels.gemm_ex(x, w, y, epi="gelu", out2=y2)),
         "resid": f / t(lambda: kernels.gemm_ex(x, w, y, epi="resid", x=y2)),
         "cublas": f / t(lambda: torch.mm(x, w.t(), out=y))}
    print(M, N, K, {k: round(v, 1) for k, v in r.items()})
