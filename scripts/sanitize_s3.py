"""Session-3 kernels under compute-sanitizer: the row-ring softmax CE (several rows per
CTA, so the 2-row ring wraps), zi_matmul_fixed through the SPEC harness, and a GPT step
with the parameter reuse cache and host-offloaded params + states."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import gpt as eg  # noqa: E402
from paper_2104_07857_b200 import harness as H  # noqa: E402
from paper_2104_07857_b200 import kernels  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402
from paper_2104_07857_b200.store import TierKind, TierStore  # noqa: E402

T, V = 300, 50304
lg = (3 * torch.randn(T, V, device="cuda")).bfloat16()
tg = torch.randint(0, V, (T,), device="cuda")
rows, loss = torch.empty(T, device="cuda"), torch.empty((), device="cuda")
kernels.softmax_ce(lg, tg, rows, loss, 1.0 / T)

L = H.LayerSpec
spec = H.ModelSpec([L("linear", 8, 16, "relu"), L("tiled_linear", 16, 16, "gelu-approx", tiles=4),
                    L("linear", 16, 4)], seed=7)
with tempfile.TemporaryDirectory() as d, TierStore(1 << 30, 1 << 30, nvme_root=d) as st:
    H.run_training(spec, 2, H.HarnessPlacement.all(TierKind.DEVICE), 3, 7, st)

c = eg.GPTConfig(nl=3, hd=128, heads=2, seq=128, vocab=256, batch=2)
pl = eg.Placement(TierKind.HOST, TierKind.HOST)
eng = eg.GPTZeroEngine(c, LocalComm(2), lr=1e-3, placement=pl, offload_chunk=10_007,
                       param_cache=1, gemm_select="zi")
for s in range(2):
    eng.step([eg.synthetic_tokens(c, 7, r, s) for r in range(2)]).item()
eng.flush()
torch.cuda.synchronize()
print("ok")
