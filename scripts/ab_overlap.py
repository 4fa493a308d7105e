"""A/B: RS + Adam on the optimizer stream (overlapped with the backward) vs on the compute
stream, graphed 1.3B steps at N=1. Prints ms/step for each, interleaved runs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import gpt as eg  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402

cfg = eg.GPT_1P3B
bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
engs = {k: eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4, overlap_opt=k)
        for k in (True, False)}
for e in engs.values():
    for s in range(3):
        e.step_graphed([bs[s % 2]])
torch.cuda.synchronize()
res = {True: [], False: []}
for rnd in range(4):
    for k, e in engs.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s in range(10):
            e.step_graphed([bs[s % 2]])
        b.record()
        torch.cuda.synchronize()
        res[k].append(a.elapsed_time(b) / 10)
print(json.dumps({"overlap_ms": [round(x, 2) for x in res[True]],
                  "serial_ms": [round(x, 2) for x in res[False]]}))
