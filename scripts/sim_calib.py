"""Simulator calibration of the optimizer-offload step: traced step vs the
lane simulator replaying its measured per-op costs. python scripts/sim_calib.py [batch]"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import gpt as eg  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402
from paper_2104_07857_b200.store import TierKind  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = dataclasses.replace(eg.GPT_1P3B, batch=batch)
eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4,
                       placement=eg.Placement(TierKind.DEVICE, TierKind.HOST))
bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
for w in range(3):
    eng.step([bs[w % 2]])
eng.trace = True
eng.step([bs[0]])
eng.flush()
torch.cuda.synchronize()
out = {"batch": batch}
for name, duplex in (("half_duplex", False), ("duplex", True)):
    sim = eng.simulated_step(duplex)
    out[name] = {k: round(sim[k], 4) for k in ("measured_s", "predicted_s", "rel_error",
                                               "forward_predicted_s", "backward_predicted_s")}
print(json.dumps(out))
