"""Diagnose AC-9 digest mismatch (tied spec): repeat runs, find first diverging step."""
import sys, os, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_07857_b200 import harness as H
from paper_2104_07857_b200.store import TierKind, TierStore
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_harness_gpu import spec
torch.backends.cuda.matmul.allow_tf32 = False
s = spec(True)
def run(world, tier, **kw):
    with tempfile.TemporaryDirectory() as d, TierStore(1 << 30, 1 << 30, nvme_root=d) as st:
        return H.run_training(s, world, H.HarnessPlacement.all(tier), 50, 7, st, **kw)
res = {}
for name, args in [("w1dev", (1, TierKind.DEVICE)), ("w1dev_b", (1, TierKind.DEVICE)),
                   ("w4nvme", (4, TierKind.NVME)), ("w4dev", (4, TierKind.DEVICE)),
                   ("w1nvme", (1, TierKind.NVME))]:
    kw = {"chunk_elems": 3} if name == "w4nvme" else {}
    res[name] = run(*args, **kw)
    print(name, res[name][0][:16], flush=True)
ref = res["w1dev"][1]
for k, (d, l) in res.items():
    first = next((i for i, (a, b) in enumerate(zip(ref, l)) if a != b), None)
    print(k, "first differing loss step vs w1dev:", first, (ref[first], l[first]) if first is not None else "")
