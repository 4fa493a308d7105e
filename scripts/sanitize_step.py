"""A tiny GPT step under compute-sanitizer: python scripts/sanitize_step.py [zi|cublas|auto]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import gpt as eg  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "zi"
c = eg.GPTConfig(nl=2, hd=128, heads=2, seq=128, vocab=256, batch=2)
eng = eg.GPTZeroEngine(c, LocalComm(2), lr=1e-3, gemm_select=mode)
for s in range(2):
    eng.step([eg.synthetic_tokens(c, 7, r, s) for r in range(2)]).item()
torch.cuda.synchronize()
print("ok", mode)
