"""zi_gemm vs cuBLAS (torch) on the GPT-1.3B step's GEMM shapes (fwd / dx / dW). One JSON line per shape."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels  # noqa: E402

T, H, V = 8192, 2048, 50304
SHAPES = [  # name, kind, M(out rows), N, K
    ("qkv.fwd", "fwd", T, 3 * H, H), ("proj.fwd", "fwd", T, H, H), ("fc1.fwd", "fwd", T, 4 * H, H),
    ("fc2.fwd", "fwd", T, H, 4 * H), ("head.fwd", "fwd", T, V, H),
    ("qkv.dx", "dx", T, H, 3 * H), ("proj.dx", "dx", T, H, H), ("fc1.dx", "dx", T, H, 4 * H),
    ("fc2.dx", "dx", T, 4 * H, H), ("head.dx", "dx", T, H, V),
    ("qkv.dW", "dw", 3 * H, H, T), ("proj.dW", "dw", H, H, T), ("fc1.dW", "dw", 4 * H, H, T),
    ("fc2.dW", "dw", H, 4 * H, T), ("head.dW", "dw32", V, H, T),
]


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    torch.manual_seed(0)
    tot_ours = tot_cub = 0.0
    for name, kind, M, N, K in SHAPES:
        bf = torch.bfloat16
        if kind == "fwd":      # y[T, out] = x[T, in] W[out, in]^T
            x = torch.randn(M, K, device="cuda", dtype=bf)
            w = torch.randn(N, K, device="cuda", dtype=bf)
            y = torch.empty(M, N, device="cuda", dtype=bf)
            ours = lambda: kernels.gemm(x, w, y)
            cub = lambda: torch.mm(x, w.t(), out=y)
        elif kind == "dx":     # dx[T, in] = dy[T, out] W[out, in]
            dy = torch.randn(M, K, device="cuda", dtype=bf)
            w = torch.randn(K, N, device="cuda", dtype=bf)
            y = torch.empty(M, N, device="cuda", dtype=bf)
            ours = lambda: kernels.gemm(dy, w.t(), y)
            cub = lambda: torch.mm(dy, w, out=y)
        else:                  # dW[out, in] = dy[T, out]^T x[T, in]
            dy = torch.randn(K, M, device="cuda", dtype=bf)
            x = torch.randn(K, N, device="cuda", dtype=bf)
            y = torch.empty(M, N, device="cuda", dtype=torch.float32 if kind == "dw32" else bf)
            ours = lambda: kernels.gemm(dy.t(), x.t(), y)
            if kind == "dw32":
                cub = lambda: y.copy_(torch.ops.aten.mm.dtype(dy.t(), x, torch.float32))
            else:
                cub = lambda: torch.mm(dy.t(), x, out=y)
        fl = 2.0 * M * N * K
        to, tc = timeit(ours), timeit(cub)
        tot_ours += to
        tot_cub += tc
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "zi_ms": round(to, 4),
                          "cublas_ms": round(tc, 4), "zi_tflops": round(fl / to / 1e9, 1),
                          "cublas_tflops": round(fl / tc / 1e9, 1)}), flush=True)
    print(json.dumps({"total_zi_ms": round(tot_ours, 3), "total_cublas_ms": round(tot_cub, 3)}))


if __name__ == "__main__":
    main()
