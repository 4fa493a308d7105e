"""Pipeline timeline of the wide-tile GEMM from clock64 stamps (zi_gemm_set_profile)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels, _lib  # noqa: E402
M, N, K = (int(v) for v in sys.argv[1:4])
epi = sys.argv[4] if len(sys.argv) > 4 else "plain"
x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
y2 = torch.empty_like(y)
args = dict(epi=epi, out2=y2 if epi == "gelu" else None, x=y2 if epi in ("resid", "dgelu") else None)
for _ in range(3):
    kernels.gemm_ex(x, w, y, **args)
prof = torch.zeros(148 * 16 * 8, dtype=torch.int64, device="cuda")
_lib.call("zi_gemm_set_profile", prof.data_ptr())
kernels.gemm_ex(x, w, y, **args)
torch.cuda.synchronize()
_lib.call("zi_gemm_set_profile", None)
p = prof.view(148, 16, 8).cpu()
import statistics as st
for cta in (0, 2, 70):
    print("cta", cta)
    for t in range(8):
        r = p[cta, t].tolist()
        if r[0] == 0:
            break
        base = p[cta, 0, 0].item()
        print(" tile", t, "mma: wait0 %d..%d wait1 %d..%d end %d | epi: seen %d h0 %d h1 %d" %
              tuple(v - base if v else -1 for v in r))
# aggregate over leader CTAs (even): mma wait for half0 / half1, epilogue drain durations
w0, w1, d0, d1, tile = [], [], [], [], []
for cta in range(0, 148, 2):
    for t in range(1, 15):
        r = p[cta, t].tolist()
        if r[0] == 0 or r[4] == 0:
            break
        w0.append(r[1] - r[0]); w1.append(r[3] - r[2])
        prev = p[cta, t - 1].tolist()
        tile.append(r[4] - prev[4])
        if prev[5] and prev[6]:
            d0.append(prev[6] - prev[5]); d1.append(prev[7] - prev[6])
f = lambda v: (round(st.mean(v)), round(st.median(v))) if v else None
print("MMA wait half0 (mean, median):", f(w0), " wait half1:", f(w1))
print("epilogue drain half0:", f(d0), " half1:", f(d1), " tile period:", f(tile))
print("ideal MMA cycles per tile:", (K // 64) * 1024)
