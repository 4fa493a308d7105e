"""compute-sanitizer target for the round-2 kernels: two GPT steps whose attention runs the
two-Q-tile forward (S = 256), the dK/dV and dQ kernels with P^T / dS^T in TMEM and the qkv
bias side output, zi_gemm_sk with preferred clusters of 4 and the gelu_save / mul / delta /
colsum epilogues; plus the split LayerNorm backward at H = 2048 (ragged T)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import gpt as eg, kernels  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402

c = eg.GPTConfig(nl=2, hd=256, heads=2, seq=256, vocab=512, batch=2)
eng = eg.GPTZeroEngine(c, LocalComm(2), lr=1e-3)
for s in range(2):
    eng.step([eg.synthetic_tokens(c, 7, r, s) for r in range(2)]).item()
T, H = 40, 2048
x = torch.randn(T, H, device="cuda").bfloat16()
w = torch.ones(H, device="cuda").bfloat16()
dy, dr = torch.randn_like(x), torch.randn_like(x)
y, mean, rstd = torch.empty_like(x), torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
kernels.ln_fwd(x, w, torch.zeros_like(w), y, mean, rstd)
g = [torch.empty(H, device="cuda") for _ in range(3)]
kernels.ln_bwd(dy, x, w, mean, rstd, torch.empty_like(x), g[0], g[1], kernels.Workspace(),
               dres=dr, dres_sum=g[2])
torch.cuda.synchronize()
print("ok")
