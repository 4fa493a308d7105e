"""Run only bench.py's NVMe optimizer-state legs (page cache and native O_DIRECT)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2104_07857_b200 import gpt as eg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nvme-dir", default=None)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
cfg = eg.GPT_1P3B
bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
print(json.dumps(bench.nvme_leg(cfg, a, bs, a.steps, direct=True)), flush=True)
