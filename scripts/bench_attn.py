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
    B, H, S, D = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (8, 16, 1024, 128)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    out = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    delta = torch.empty_like(lse)
    dout = torch.randn_like(out)
    dqkv = torch.empty_like(qkv)
    unit = 2.0 * B * H * S * S * D / 2      # one causal matmul
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
