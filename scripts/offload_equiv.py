"""Run only bench.py's config-balance offload leg (one JSON line).
python scripts/offload_equiv.py [--batch 64] [--params-host]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--params-host", action="store_true")
a = ap.parse_args()
print(json.dumps(bench.offload_equiv_leg(a, a.batch, a.params_host)), flush=True)
