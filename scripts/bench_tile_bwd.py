"""The config-4 tile backward GEMMs (T=8): dW_t = g_t^T x and dx += g_t W_t, zi vs cuBLAS."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import kernels  # noqa: E402

M, K, Nt = 8192, 16384, 8192
x = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(Nt, K, device="cuda") * K ** -0.5).bfloat16()
g = (torch.randn(M, 65536, device="cuda") * 1e-2).bfloat16()[:, :Nt]
dw = torch.empty(Nt, K, device="cuda", dtype=torch.bfloat16)
dx = torch.zeros(M, K, device="cuda")
dxb = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


fl = 2.0 * M * K * Nt
gc = g.contiguous()
for name, fn in (("dW zi", lambda: kernels.gemm(g.t(), x.t(), dw)),
                 ("dW cublas", lambda: torch.mm(g.t(), x, out=dw)),
                 ("dx+= zi f32", lambda: kernels.gemm(g, W.t(), dx, accumulate=True)),
                 ("dx zi bf16", lambda: kernels.gemm(g, W.t(), dxb)),
                 ("dx cublas bf16", lambda: torch.mm(gc, W, out=dxb)),
                 ("dx+= cublas f32", lambda: dx.add_(torch.mm(gc, W, out_dtype=torch.float32)))):
    try:
        ms = t(fn)
        print(json.dumps({"gemm": name, "ms": round(ms, 3), "tflops": round(fl / ms / 1e9, 1)}))
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"gemm": name, "error": repr(e)[:120]}))
