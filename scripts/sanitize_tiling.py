"""A small config-4-shaped tiled linear (forward + backward on tcgen05) and the fused
LayerNorm / bias-grad / cross-entropy kernels, for compute-sanitizer runs."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import kernels  # noqa: E402
from paper_2104_07857_b200.store import TierKind, TierStore  # noqa: E402
from paper_2104_07857_b200.tiling import backward_tiled, forward_tiled, tile_linear  # noqa: E402

M, K, N = 512, 1024, 4096
x = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(N, K, device="cuda") * K ** -0.5).bfloat16()
b = torch.randn(N, device="cuda").bfloat16()
with TierStore(1 << 30, 1 << 28, nvme_root=tempfile.mkdtemp()) as st:
    tl = tile_linear(W, b, 4, st, TierKind.DEVICE, key="s")
    y = forward_tiled(tl, x, st)
    backward_tiled(tl, x, torch.randn(M, N, device="cuda").bfloat16(), st)
y2 = torch.empty(M, 512, device="cuda", dtype=torch.bfloat16)
kernels.gemm_ex(x, W[:512], y2, bias=b[:512], epi="gelu", out2=torch.empty_like(y2))
torch.cuda.synchronize()
print("ok")
