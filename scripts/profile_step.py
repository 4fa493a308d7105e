"""One GPT-1.3B engine step inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off ...` launch lists (exactly one step's kernels)."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2104_07857_b200 import gpt as eg  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nl", type=int, default=None)
ap.add_argument("--graph", action="store_true")
a = ap.parse_args()
cfg = eg.GPT_1P3B if a.nl is None else eg.GPTConfig(**{**eg.GPT_1P3B.__dict__, "nl": a.nl})
eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4)
bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
run = eng.step_graphed if a.graph else eng.step
for s in range(3):
    run([bs[s % 2]])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
run([bs[0]])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
