"""Stream-K GEMM (zi_gemm_sk, split and whole-tile) vs cuBLAS vs zi_gemm at the GPT-1.3B
step's 15 GEMM sites, with the sites' fused epilogues. One JSON line per site, then totals
(per step: x24 blocks for block sites). CUDA-event timing, warm, interleaved rounds, best of."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels  # noqa: E402

T, H, V = 8192, 2048, 50304
bf = torch.bfloat16


def timeit(fn, iters=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def rnd(*s, scale=1.0):
    return (torch.randn(*s, device="cuda") * scale).to(bf)


def sites():
    H3, H4 = 3 * H, 4 * H
    x, u, x2 = rnd(T, H), rnd(T, H4), rnd(T, H)
    w3, w1, w2, wp = rnd(H3, H, scale=0.02), rnd(H4, H, scale=0.02), rnd(H, H4, scale=0.02), rnd(H, H, scale=0.02)
    b3, b1, bh = rnd(H3), rnd(H4), rnd(H)
    o3, o4, oh, a4 = (torch.empty(T, n, dtype=bf, device="cuda") for n in (H3, H4, H, H4))
    g3, g1, g2, gp = (torch.empty_like(w) for w in (w3, w1, w2, wp))
    dy3, dy4 = rnd(T, H3), rnd(T, H4)
    wte = rnd(V, H, scale=0.02)
    logits = torch.empty(T, V, dtype=bf, device="cuda")
    acc = torch.empty(V, H, dtype=torch.float32, device="cuda")
    dx = torch.empty(T, H, dtype=bf, device="cuda")
    S = []

    def site(name, n, M, N, K, sk, cub, zi=None):
        S.append((name, n, 2.0 * M * N * K, sk, cub, zi))

    site("qkv.fwd", 24, T, H3, H, lambda s: kernels.gemm_sk(x, w3, o3, bias=b3, split=s),
         lambda: torch.addmm(b3, x, w3.t(), out=o3), lambda: kernels.gemm(x, w3, o3, bias=b3))
    site("proj.fwd", 24, T, H, H, lambda s: kernels.gemm_sk(x, wp, oh, bias=bh, split=s),
         lambda: torch.addmm(bh, x, wp.t(), out=oh), lambda: kernels.gemm(x, wp, oh, bias=bh))
    site("fc1.fwd+gelu", 24, T, H4, H,
         lambda s: kernels.gemm_sk(x, w1, o4, bias=b1, epi="gelu", out2=a4, split=s),
         lambda: (torch.addmm(b1, x, w1.t(), out=o4), kernels.gelu_fwd(o4, a4)),
         lambda: kernels.gemm_ex(x, w1, o4, bias=b1, epi="gelu", out2=a4))
    site("fc2.fwd+resid", 24, T, H, H4,
         lambda s: kernels.gemm_sk(u, w2, oh, bias=bh, epi="resid", x=x2, split=s),
         lambda: (torch.addmm(bh, u, w2.t(), out=oh), oh.add_(x2)),
         lambda: kernels.gemm_ex(u, w2, oh, bias=bh, epi="resid", x=x2))
    site("fc2.dW", 24, H, H4, T, lambda s: kernels.gemm_sk(x.t(), u.t(), g2, split=s),
         lambda: torch.mm(x.t(), u, out=g2), lambda: kernels.gemm(x.t(), u.t(), g2))
    site("fc1.dW", 24, H4, H, T, lambda s: kernels.gemm_sk(dy4.t(), x.t(), g1, split=s),
         lambda: torch.mm(dy4.t(), x, out=g1), lambda: kernels.gemm(dy4.t(), x.t(), g1))
    site("proj.dW", 24, H, H, T, lambda s: kernels.gemm_sk(x.t(), x2.t(), gp, split=s),
         lambda: torch.mm(x.t(), x2, out=gp), lambda: kernels.gemm(x.t(), x2.t(), gp))
    site("qkv.dW", 24, H3, H, T, lambda s: kernels.gemm_sk(dy3.t(), x.t(), g3, split=s),
         lambda: torch.mm(dy3.t(), x, out=g3), lambda: kernels.gemm(dy3.t(), x.t(), g3))
    site("fc2.dx+dgelu", 24, T, H4, H,
         lambda s: kernels.gemm_sk(x, w2.t(), a4, epi="dgelu", x=u, split=s),
         lambda: torch.mm(x, w2, out=o4),
         lambda: kernels.gemm_ex(x, w2.t(), a4, epi="dgelu", x=u))
    site("fc1.dx", 24, T, H, H4, lambda s: kernels.gemm_sk(dy4, w1.t(), oh, split=s),
         lambda: torch.mm(dy4, w1, out=oh), lambda: kernels.gemm(dy4, w1.t(), oh))
    site("proj.dx", 24, T, H, H, lambda s: kernels.gemm_sk(x2, wp.t(), oh, split=s),
         lambda: torch.mm(x2, wp, out=oh), lambda: kernels.gemm(x2, wp.t(), oh))
    site("qkv.dx", 24, T, H, H3, lambda s: kernels.gemm_sk(dy3, w3.t(), oh, split=s),
         lambda: torch.mm(dy3, w3, out=oh), lambda: kernels.gemm(dy3, w3.t(), oh))
    site("head.fwd", 1, T, V, H, lambda s: kernels.gemm_sk(x, wte, logits, split=s),
         lambda: torch.mm(x, wte.t(), out=logits), lambda: kernels.gemm(x, wte, logits))
    site("head.dW", 1, V, H, T, lambda s: kernels.gemm_sk(logits.t(), x.t(), acc, split=s),
         lambda: torch.ops.aten.mm.dtype_out(logits.t(), x, torch.float32, out=acc),
         lambda: kernels.gemm(logits.t(), x.t(), acc))
    site("head.dx", 1, T, H, V, lambda s: kernels.gemm_sk(logits, wte.t(), dx, split=s),
         lambda: torch.mm(logits, wte, out=dx), lambda: kernels.gemm(logits, wte.t(), dx))
    return S


def main():
    torch.manual_seed(0)
    only = sys.argv[1:] or None
    tot = {"sk": 0.0, "whole": 0.0, "cublas": 0.0, "zi": 0.0, "best_lib": 0.0}
    for name, n, fl, sk, cub, zi in sites():
        if only and name not in only:
            continue
        cands = {"sk": lambda: sk(True), "whole": lambda: sk(False), "cublas": cub, "zi": zi}
        for f in cands.values():
            f()
        torch.cuda.synchronize()
        best = {k: 1e9 for k in cands}
        for _ in range(3):
            for k, f in cands.items():
                best[k] = min(best[k], timeit(f))
        row = {"site": name, "per_step": n}
        for k in cands:
            row[k + "_ms"] = round(best[k], 4)
            row[k + "_tflops"] = round(fl / best[k] / 1e9, 1)
            tot[k] += best[k] * n
        tot["best_lib"] += min(best["cublas"], best["zi"]) * n
        print(json.dumps(row), flush=True)
    print(json.dumps({"per_step_ms": {k: round(v, 3) for k, v in tot.items()}}))


if __name__ == "__main__":
    main()
