"""A/B of the params+optimizer offload step at config-5 balance (1.3B x 32 seq/GPU):
forward-interleaved optimizer-state prefetch (every k blocks) x staging-ring depth.
python scripts/ab_config5.py [k:slots ...]"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import gpt as eg  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402
from paper_2104_07857_b200.store import TierKind  # noqa: E402

cfg = dataclasses.replace(eg.GPT_1P3B, batch=int(os.environ.get("BATCH", 32)))
bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
H = TierKind.HOST
for v in (sys.argv[1:] or ["0:12", "3:12", "2:12", "3:16"]):
    k, ns = (int(x) for x in v.split(":"))
    eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4, placement=eg.Placement(H, H),
                           offload_slots=ns, fwd_state_prefetch_every=k,
                           param_cache=int(os.environ.get("CACHE", 0)))
    for w in range(2):
        eng.step([bs[w % 2]])
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in range(3):
        loss = eng.step([bs[s % 2]])
    eng.flush()
    t1.record()
    torch.cuda.synchronize()
    eng.trace = True
    eng.step([bs[0]])
    tl = eng.timeline()
    eng.trace = False
    print(json.dumps({"every": k, "slots": ns, "ms": round(t0.elapsed_time(t1) / 3, 2),
                      "loss": float(loss.item()), "pcie_busy_s": round(tl.lane_busy_s("pcie"), 4),
                      "tl_hidden": round(tl.hidden_fraction(("pcie",)), 4)}), flush=True)
    del eng
    torch.cuda.empty_cache()
