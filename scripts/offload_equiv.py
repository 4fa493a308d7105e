"""Run only bench.py's config-3-equivalent optimizer-offload leg (one JSON line)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
print(json.dumps(bench.offload_equiv_leg(a, a.batch)), flush=True)
