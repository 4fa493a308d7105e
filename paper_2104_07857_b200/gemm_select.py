"""zi_gemm_sk vs cuBLAS on the GPT step's linears: the A/B comparison behind the bench's
``gemm_sites`` column (and the engine's opt-in ``gemm_select="auto"`` mode).

Each linear of the block and the head is one *site*. The product path runs every site on
zi_gemm_sk (tcgen05 stream-K; the neighbouring elementwise pass folded into its epilogue
where the site has one: bias + GELU, bias + residual, GELU' for the fc1 gradient). The
cuBLAS candidate computes the same outputs with the pass as a separate libzinf / torch
kernel. ``tune`` times both on the site's real shapes with CUDA events (interleaved, best
of several) once per process and caches the result.

``ZI_GEMM_SELECT`` = ``zi`` (default) | ``cublas`` | ``auto`` forces a choice.
"""

from __future__ import annotations

import os

import torch

from . import kernels

_CHOICE: dict = {}          # (site, shape...) -> "zi" | "cublas"
_TIMES: dict = {}           # same key -> (zi_ms, cublas_ms), for reports
_REPORT = False             # compare_gpt: time both candidates whatever the mode


def aligned(*ts) -> bool:
    """zi_gemm's operand contract: 16-byte aligned bases; a 2-D operand has one unit
    stride and the other a multiple of 8 elements."""
    for t in ts:
        if t is None:
            continue
        if t.data_ptr() % 16:
            return False
        if t.dim() == 2:
            s0, s1 = t.stride()
            if not ((s1 == 1 and s0 % 8 == 0) or (s0 == 1 and s1 % 8 == 0)):
                return False
    return True


def _time(fn, reps: int) -> float:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def tune(key, zi_fn, cublas_fn, rounds: int = 3, reps: int = 5) -> str:
    mode = os.environ.get("ZI_GEMM_SELECT", "auto")
    if mode in ("zi", "cublas") and not _REPORT:
        return mode
    if key in _CHOICE:
        return _CHOICE[key]
    for fn in (zi_fn, cublas_fn):   # warm: plans, TMA descriptors, caches
        fn()
    torch.cuda.synchronize()
    tz, tc = [], []
    for _ in range(rounds):         # interleaved so clock drift hits both alike
        tz.append(_time(zi_fn, reps))
        tc.append(_time(cublas_fn, reps))
    z, c = min(tz), min(tc)
    _CHOICE[key] = "zi" if z < c else "cublas"
    _TIMES[key] = (round(z, 4), round(c, 4))
    return _CHOICE[key]


def compare_gpt(T: int, hd: int, vocab: int, ws, device) -> dict:
    """Time zi_gemm_sk against cuBLAS at every site (the bench's comparison column);
    returns :func:`report`."""
    global _REPORT
    _REPORT = True
    try:
        tune_gpt(T, hd, vocab, ws, device)
    finally:
        _REPORT = False
    return report()


def report() -> dict:
    """{site: {"choice", "zi_ms", "cublas_ms"}} of every tuned site in this process."""
    return {"/".join(str(k) for k in key): {"choice": _CHOICE[key], "zi_ms": t[0],
                                             "cublas_ms": t[1]}
            for key, t in _TIMES.items()}


def tune_gpt(T: int, hd: int, vocab: int, ws, device) -> dict:
    """Choose every site of the GPT block and the tied head at T tokens x hidden hd.

    Returns {site: "zi" | "cublas"}. Dummy operands of the exact shapes; each candidate
    computes the site's full output set.
    """
    bf = torch.bfloat16
    g = torch.Generator(device=device).manual_seed(0)

    def rnd(*shape, scale=0.05):
        return (torch.randn(*shape, device=device, generator=g) * scale).to(bf)

    H3, H4 = 3 * hd, 4 * hd
    x, u = rnd(T, hd), rnd(T, H4)
    w3, w1, w2, wp = rnd(H3, hd), rnd(H4, hd), rnd(hd, H4), rnd(hd, hd)
    b3, b1, bh = rnd(H3), rnd(H4), rnd(hd)
    o3, o4, oh, oh2 = (torch.empty(T, n, dtype=bf, device=device) for n in (H3, H4, hd, hd))
    a4 = torch.empty(T, H4, dtype=bf, device=device)
    gw3, gw1, gw2, gwp = (torch.empty_like(w) for w in (w3, w1, w2, wp))
    db = torch.empty(H4, dtype=bf, device=device)
    dy4 = rnd(T, H4)
    dy3 = rnd(T, H3)
    sites = {}
    # forward: qkv / proj (bias), fc1 (+ GELU), fc2 (+ bias + residual)
    for name, w, b, out in (("qkv.fwd", w3, b3, o3), ("proj.fwd", wp, bh, oh)):
        sites[name] = tune((name, T, w.shape[0], hd),
                           lambda w=w, b=b, out=out: kernels.gemm_sk(x, w, out, bias=b),
                           lambda w=w, b=b, out=out: torch.addmm(b, x, w.t(), out=out))
    # the product path's epilogues: fc1 keeps GELU' for the backward ("gelu_save"), fc2.dx
    # multiplies by it and sums the fc1 bias gradient's 32-row blocks (+ the fold)
    sites["fc1.fwd"] = tune(("fc1.fwd+gelu", T, H4, hd),
                            lambda: kernels.gemm_sk(x, w1, o4, bias=b1, epi="gelu_save", out2=a4),
                            lambda: (torch.addmm(b1, x, w1.t(), out=o4), kernels.gelu_fwd(o4, a4)))
    sites["fc2.fwd"] = tune(("fc2.fwd+resid", T, hd, H4),
                            lambda: kernels.gemm_sk(u, w2, oh, bias=bh, epi="resid", x=oh2),
                            lambda: (torch.addmm(bh, u, w2.t(), out=oh), oh.add_(oh2)))
    # backward: weight gradients (both operands MN-major) and input gradients
    for name, dy, inp, gw in (("fc2.dW", x, u, gw2), ("fc1.dW", dy4, x, gw1),
                              ("proj.dW", x, x, gwp), ("qkv.dW", dy3, x, gw3)):
        sites[name] = tune((name, T, gw.shape[0], gw.shape[1]),
                           lambda dy=dy, inp=inp, gw=gw: kernels.gemm_sk(dy.t(), inp.t(), gw),
                           lambda dy=dy, inp=inp, gw=gw: torch.mm(dy.t(), inp, out=gw))
    part = torch.empty(-(-T // 32) * H4, dtype=torch.float32, device=device)
    sites["fc2.dx"] = tune(("fc2.dx+dgelu", T, H4, hd),
                           lambda: (kernels.gemm_sk(x, w2.t(), a4, epi="mul", x=u, colsum=part),
                                    kernels.colsum_fold(part, -(-T // 32), H4, db)),
                           lambda: (torch.mm(x, w2, out=o4), kernels.bias_grad(o4, db, ws, u=u,
                                                                                du=a4)))
    for name, dy, w, out in (("fc1.dx", dy4, w1, oh), ("proj.dx", x, wp, oh),
                             ("qkv.dx", dy3, w3, oh)):
        sites[name] = tune((name, T, hd, dy.shape[1]),
                           lambda dy=dy, w=w, out=out: kernels.gemm_sk(dy, w.t(), out),
                           lambda dy=dy, w=w, out=out: torch.mm(dy, w, out=out))
    del x, u, w3, w1, w2, wp, o3, o4, oh, oh2, a4, gw3, gw1, gw2, gwp, dy4, dy3, part
    # tied head: logits, dW (fp32 accumulator), dx
    hf, wte = rnd(T, hd), rnd(vocab, hd)
    logits = torch.empty(T, vocab, dtype=bf, device=device)
    acc = torch.empty(vocab, hd, dtype=torch.float32, device=device)
    dx = torch.empty(T, hd, dtype=bf, device=device)
    sites["head.fwd"] = tune(("head.fwd", T, vocab, hd),
                             lambda: kernels.gemm_sk(hf, wte, logits),
                             lambda: torch.mm(hf, wte.t(), out=logits))
    sites["head.dW"] = tune(("head.dW", vocab, hd, T),
                            lambda: kernels.gemm_sk(logits.t(), hf.t(), acc),
                            lambda: torch.ops.aten.mm.dtype_out(logits.t(), hf, torch.float32,
                                                                out=acc))
    sites["head.dx"] = tune(("head.dx", T, hd, vocab),
                            lambda: kernels.gemm_sk(logits, wte.t(), dx),
                            lambda: torch.mm(logits, wte, out=dx))
    del hf, wte, logits, acc, dx
    torch.cuda.synchronize()
    return sites
