"""BASELINE config 4: memory-centric tiling of one 16384 -> 65536 linear into T = 4/8/16 tiles.

python bench_tiling.py [--tokens 8192] [--iters 5]

Per T: forward_tiled through the partitioned tier store (N=1: each tile's
shard is the whole tile, gathered just in time into a 2-slot ring on a
side stream) with every tile product on zi_linear_fwd (tcgen05). Reports
TFLOPS = 2*M*K*N / t against the measured bf16 peak, next to cuBLAS
(torch.addmm) on the same tiles. One JSON line per T.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tiles", default="4,8,16")
    args = ap.parse_args()
    from bench import _peaks
    from paper_2104_07857_b200 import kernels
    from paper_2104_07857_b200.store import TierKind, TierStore
    from paper_2104_07857_b200.tiling import forward_tiled, tile_linear

    torch.cuda.set_device(0)
    M, K, N = args.tokens, 16384, 65536
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    W = (torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * K ** -0.5)
    b = torch.randn(N, device="cuda", dtype=torch.bfloat16, generator=g)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    _, peak, kind = _peaks()
    flops = 2.0 * M * K * N
    for T in [int(t) for t in args.tiles.split(",")]:
        with TierStore(16 << 30, 1 << 30, nvme_root=tempfile.mkdtemp()) as st:
            tl = tile_linear(W, b, T, st, TierKind.DEVICE, key=f"fc{T}")

            def ours():
                forward_tiled(tl, x, st, out=y)

            def cublas():
                for s, e in tl.rows:
                    torch.addmm(b[s:e], x, W[s:e].t(), out=y[:, s:e]) if False else \
                        y[:, s:e].copy_(torch.addmm(b[s:e], x, W[s:e].t()))

            res = {}
            for name, fn in (("tcgen05", ours), ("cublas", cublas)):
                for _ in range(args.warmup):
                    fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.iters):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.iters
                res[name] = (ms, flops / (ms / 1e3) / 1e12)
            # single-tile kernel timing (no gather), for the roofline
            s0, e0_ = tl.rows[0]
            Wt = W[s0:e0_]
            yt = y[:, s0:e0_]
            for _ in range(3):
                kernels.linear_fwd(x, Wt, b[s0:e0_], yt)
            torch.cuda.synchronize()
            a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.iters):
                kernels.linear_fwd(x, Wt, b[s0:e0_], yt)
            c.record()
            torch.cuda.synchronize()
            kms = a.elapsed_time(c) / args.iters
            ktf = 2.0 * M * K * (e0_ - s0) / (kms / 1e3) / 1e12
            ref = (x[:256].float() @ W[:4096].float().t() + b[:4096].float())
            forward_tiled(tl, x, st, out=y)
            err = ((y[:256, :4096].float() - ref).abs() / (ref.abs() + 1e-2)).max().item()
            print(json.dumps({
                "workload": f"tiled linear 16384->65536, T={T}, M={M} tokens, bf16",
                "tiles": T, "tile_rows": tl.rows[0][1] - tl.rows[0][0],
                "forward_tiled_ms": round(res["tcgen05"][0], 3),
                "forward_tiled_tflops": round(res["tcgen05"][1], 1),
                "cublas_same_tiles_ms": round(res["cublas"][0], 3),
                "cublas_tflops": round(res["cublas"][1], 1),
                "tile_kernel_tflops": round(ktf, 1),
                "roofline": {"bound": "tensor", "achieved": round(ktf, 1), "peak": peak,
                             "peak_kind": kind, "unit": "TFLOP/s", "frac": round(ktf / peak, 4)},
                "max_rel_err_vs_fp32": round(err, 5),
            }), flush=True)


if __name__ == "__main__":
    main()
