"""One GEMM shape on zi_gemm_sk (split, then whole tiles) then cuBLAS, for ncu:
python scripts/gemm_sk_one.py M N K [fwd|dx|dw]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels  # noqa: E402
M, N, K = (int(v) for v in sys.argv[1:4])
kind = sys.argv[4] if len(sys.argv) > 4 else "fwd"
bf = torch.bfloat16
if kind == "fwd":
    a, b = torch.randn(M, K, device="cuda", dtype=bf), torch.randn(N, K, device="cuda", dtype=bf)
elif kind == "dx":
    a, b = torch.randn(M, K, device="cuda", dtype=bf), torch.randn(K, N, device="cuda", dtype=bf).t()
else:
    a, b = torch.randn(K, M, device="cuda", dtype=bf).t(), torch.randn(K, N, device="cuda", dtype=bf).t()
y = torch.empty(M, N, device="cuda", dtype=bf)
for _ in range(3):
    kernels.gemm_sk(a, b, y, split=True)
    kernels.gemm_sk(a, b, y, split=False)
    torch.mm(a, b.t(), out=y)
torch.cuda.synchronize()
