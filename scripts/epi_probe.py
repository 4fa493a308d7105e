"""zi_gemm_sk epilogue cost at the fc2.dx site (8192 x 8192 x 2048, B MN-major): plain vs
GELU' (reads the pre-activation) vs GELU' + fc1 bias column sums. Warm CUDA-event timing,
interleaved rounds, best of 3."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels  # noqa: E402

M, N, K = 8192, 8192, 2048
bf = torch.bfloat16
a = torch.randn(M, K, device="cuda", dtype=bf)
w = (torch.randn(K, N, device="cuda") * K ** -0.5).to(bf)
b = w.t()
u = torch.randn(M, N, device="cuda", dtype=bf)
y = torch.empty(M, N, device="cuda", dtype=bf)
part = torch.empty(M // 32 * N, device="cuda")
cases = {
    "plain": lambda: kernels.gemm_sk(a, b, y),
    "dgelu": lambda: kernels.gemm_sk(a, b, y, epi="dgelu", x=u),
    "dgelu+colsum": lambda: kernels.gemm_sk(a, b, y, epi="dgelu", x=u, colsum=part),
    "mul+colsum": lambda: kernels.gemm_sk(a, b, y, epi="mul", x=u, colsum=part),
}
# the fc1 forward site (8192 x 8192 x 2048, K-major B): GELU vs GELU'-saving epilogue
h = torch.randn(M, K, device="cuda", dtype=bf)
w1 = (torch.randn(N, K, device="cuda") * K ** -0.5).to(bf)
b1 = torch.randn(N, device="cuda", dtype=bf)
y2 = torch.empty(M, N, device="cuda", dtype=bf)
cases["fwd gelu"] = lambda: kernels.gemm_sk(h, w1, y, bias=b1, epi="gelu", out2=y2)
cases["fwd gelu_save"] = lambda: kernels.gemm_sk(h, w1, y, bias=b1, epi="gelu_save", out2=y2)


def t(fn, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for f in cases.values():
    f()
torch.cuda.synchronize()
best = {k: 1e9 for k in cases}
for _ in range(3):
    for k, f in cases.items():
        best[k] = min(best[k], t(f))
for k, v in best.items():
    print(f"{k:14s} {v * 1e3:7.1f} us  {2 * M * N * K / v / 1e9:7.1f} TFLOPS")
