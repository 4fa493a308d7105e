"""One wide-tile gemm_ex launch (for ncu): python scripts/gemm_one_ex.py M N K [epi]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels  # noqa: E402
M, N, K = (int(v) for v in sys.argv[1:4])
epi = sys.argv[4] if len(sys.argv) > 4 else "plain"
x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
y2 = torch.empty_like(y)
for _ in range(3):
    kernels.gemm_ex(x, w, y, epi=epi, out2=y2 if epi == "gelu" else None,
                    x=y2 if epi in ("resid", "dgelu") else None)
torch.cuda.synchronize()
