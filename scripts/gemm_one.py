"""One GEMM shape, ours then cuBLAS (for ncu): python scripts/gemm_one.py M N K [kind]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels  # noqa: E402
M, N, K = (int(v) for v in sys.argv[1:4])
kind = sys.argv[4] if len(sys.argv) > 4 else "fwd"
x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    kernels.gemm(x, w, y)
    torch.mm(x, w.t(), out=y)
torch.cuda.synchronize()
