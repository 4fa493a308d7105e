"""Time zi_attn_fwd / zi_attn_bwd against cuDNN/flash SDPA (torch) at the 1.3B block shape.

Usage: python scripts/bench_attn.py [B H S D]. TFLOPS count executed causal work:
fwd 2 matmuls, bwd 5 (dK/dV + dQ kernels recompute S and dP: 7 executed), each
2*B*H*S*S*D/2 flops.
"""
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2104_07857_b200 import kernels  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    once = "--once" in sys.argv
    argv = [a for a in sys.argv[1:] if a != "--once"]
    B, H, S, D = (int(x) for x in argv[:4]) if len(argv) >= 4 else (8, 16, 1024, 128)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    out = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    delta = torch.empty_like(lse)
    dout = torch.randn_like(out)
    dqkv = torch.empty_like(qkv)
    unit = 2.0 * B * H * S * S * D / 2      # one causal matmul
    if "--trace-bwd" in sys.argv:           # CTA 0 of the dK / dV kernel (j = 0: 16 sub-tiles)
        from paper_2104_07857_b200 import _lib
        kernels.attn_fwd(qkv, out, lse, B, H)
        tr = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
        _lib.call("zi_attn_set_trace", tr.data_ptr())
        kernels.attn_bwd(qkv, out, dout, lse, delta, dqkv, B, H)
        torch.cuda.synchronize()
        _lib.call("zi_attn_set_trace", None)
        t = tr.view(64, 8).cpu().double()
        base = t[0, 0]
        print("u: [S qd landed, st_free, S issued | acc ps_full | group st_full, ps_empty, published] kcycles")
        for u in range(2 * (S // 128)):
            print("   ", u, [round(float(v - base) / 1000, 2) for v in t[u, :7]])
        return
    if "--trace2" in sys.argv:              # per-CTA timeline of the two-q-tile forward
        from paper_2104_07857_b200 import _lib
        nct = B * H * (S // 256)
        tr = torch.zeros(nct * 6 + 3 * 16 * 4, dtype=torch.int64, device="cuda")
        kernels.attn_fwd(qkv, out, lse, B, H)
        torch.cuda.synchronize()
        _lib.call("zi_attn_set_trace", tr.data_ptr())
        kernels.attn_fwd(qkv, out, lse, B, H)
        torch.cuda.synchronize()
        _lib.call("zi_attn_set_trace", None)
        t = tr[:nct * 6].view(nct, 6).cpu().double()
        fine = tr[nct * 6:].view(3, 16, 4).cpu().double()
        t0 = t[:, 1].min()
        t[:, 1:] = (t[:, 1:] - t0) / 1000.0
        print("kernel span us", float(t[:, 5].max()))
        for name, a, b in (("entry->operands", 1, 2), ("operands->last mma", 2, 3),
                           ("last mma->softmax b done", 3, 4), ("softmax b done->exit", 4, 5),
                           ("cta total", 1, 5)):
            d = t[:, b] - t[:, a]
            print(f"{name:26s} mean {float(d.mean()):6.2f} us  max {float(d.max()):6.2f}")
        base = fine[0, 0, 0]
        nkvb = S // 128                       # CTA 0 = the last q tile pair
        for x in range(2):
            print(f"group {x}: [wait start, S ready, max done, P published] kcycles")
            for j in range(nkvb - 1 + x):
                print("   ", j, [round(float(v - base) / 1000, 2) for v in fine[x, j]])
        print("MMA: [PV_a, S_a(j+1), PV_b, S_b(j+1)] issued, kcycles")
        for j in range(nkvb):
            print("   ", j, [round(float(v - base) / 1000, 2) if v > 0 else None for v in fine[2, j]])
        return
    if "--trace" in sys.argv:               # per-CTA timeline of the forward
        from paper_2104_07857_b200 import _lib
        nct = B * H * (S // 128)
        tr = torch.zeros(nct * 6 + 2 * 64 * 6 + 32 * 4, dtype=torch.int64, device="cuda")
        kernels.attn_fwd(qkv, out, lse, B, H)
        torch.cuda.synchronize()
        _lib.call("zi_attn_set_trace", tr.data_ptr())
        kernels.attn_fwd(qkv, out, lse, B, H)
        torch.cuda.synchronize()
        _lib.call("zi_attn_set_trace", None)
        fine = tr[nct * 6:nct * 6 + 768].view(2, 64, 6).cpu().double()
        mm = tr[nct * 6 + 768:].view(32, 4).cpu().double()
        t = tr[:nct * 6].view(nct, 6).cpu().double()
        t0 = t[:, 1].min()
        t[:, 1:] -= t0
        t[:, 1:] /= 1000.0
        print("kernel span us", float(t[:, 5].max()))
        for name, a, b in (("entry->operands", 1, 2), ("operands->last mma", 2, 3),
                           ("last mma->softmax done", 3, 4), ("softmax done->exit", 4, 5),
                           ("cta total", 1, 5)):
            d = t[:, b] - t[:, a]
            print(f"{name:24s} mean {float(d.mean()):6.2f} us  max {float(d.max()):6.2f}")
        # gaps between consecutive CTAs on one SM
        gaps = []
        for sm in t[:, 0].unique():
            rows = t[t[:, 0] == sm]
            rows = rows[rows[:, 1].argsort()]
            gaps += (rows[1:, 1] - rows[:-1, 5]).tolist()
        g = torch.tensor(gaps)
        print(f"inter-CTA gap on an SM: mean {float(g.mean()):.2f} us max {float(g.max()):.2f}; "
              f"CTAs per SM {nct / t[:, 0].unique().numel():.1f}")
        for g in range(2):
            f = fine[g]
            base = f[0, 0]
            print(f"group {g} sub-tiles of CTA 0 (kcycles from its first wait): "
                  "[start, S ready, S loaded, exps done, pv waited, P published]")
            for jj in range(S // 128):
                print("   ", [round(float(x - base) / 1000, 2) for x in f[jj]])
        base = fine[0, 0, 0]
        print("MMA thread of CTA 0 per u: [loop top, kv landed, s_free, p_full(u-1)] kcycles")
        for u in range(2 * (S // 128) + 1):
            print("   ", u, [round(float(x - base) / 1000, 2) if x > 0 else None for x in mm[u]])
        for nkv in (1, 4, 8):
            rows = t[(torch.arange(nct) // (B * H)) == (S // 128 - nkv)]
            print(f"  nkv={nkv}: cta {float((rows[:, 5] - rows[:, 1]).mean()):.2f} us, "
                  f"mma {float((rows[:, 3] - rows[:, 2]).mean()):.2f} us")
        return
    if once:                                 # one launch of each kernel (for ncu)
        kernels.attn_fwd(qkv, out, lse, B, H)
        kernels.attn_bwd(qkv, out, dout, lse, delta, dqkv, B, H)
        torch.cuda.synchronize()
        return
    t_f = timeit(lambda: kernels.attn_fwd(qkv, out, lse, B, H))
    t_b = timeit(lambda: kernels.attn_bwd(qkv, out, dout, lse, delta, dqkv, B, H))
    leaf = qkv.detach().requires_grad_(True)
    q, k, v = leaf.view(B, S, 3, H, D).unbind(2)
    q, k, v = (t.transpose(1, 2) for t in (q, k, v))

    def sdpa_f():
        return F.scaled_dot_product_attention(q, k, v, is_causal=True)
    o4 = sdpa_f()
    g4 = dout.view(B, S, H, D).transpose(1, 2)
    c_f = timeit(sdpa_f)
    c_b = timeit(lambda: torch.autograd.grad(o4, leaf, g4, retain_graph=True))
    print(f"shape B{B} H{H} S{S} D{D}")
    print(f"zi   fwd {t_f:.3f} ms ({2 * unit / t_f / 1e9:.0f} TF exec)  bwd {t_b:.3f} ms "
          f"({7 * unit / t_b / 1e9:.0f} TF exec, {5 * unit / t_b / 1e9:.0f} TF model)")
    print(f"sdpa fwd {c_f:.3f} ms ({2 * unit / c_f / 1e9:.0f} TF)       bwd {c_b:.3f} ms "
          f"({5 * unit / c_b / 1e9:.0f} TF model)")


if __name__ == "__main__":
    main()
