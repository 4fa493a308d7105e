"""Regenerate tests/golden/planner_ref.json from the REFERENCE memory / efficiency models.

``planner.py`` restates the reference's closed-form sizing and bandwidth formulas
(``memory.py:83-121``, ``efficiency.py:38-90``). This script imports the reference
``infinisim.memory`` / ``infinisim.efficiency`` (from /root/reference/pkg/src — build
container only) and records their outputs on a grid of shapes, so the planner is pinned
to the reference's own numbers on the GPU box too (tests/test_planner.py).

Usage: python tests/golden/make_planner_golden.py
"""

from __future__ import annotations

import itertools
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

SHAPES = [dict(nl=nl, hd=hd, attn_heads=ah, seq=seq, bsz=bsz, ci=ci)
          for nl, hd, ah, seq, bsz, ci in itertools.product(
              (1, 24, 50, 125), (256, 2048, 4096, 8192, 25600), (4, 32), (128, 1024),
              (0.25, 1, 8, 1.25), (1, 4))
          if ci <= nl]
BWS = (1e6, 3e9, 12e9, 48e9, 1.5e12, 7.7e12, float("inf"))
PEAKS = (70e12, 2.25e15)
EFFS = (0.1, 0.5, 0.9, 0.99)


def main(out=os.path.join(HERE, "planner_ref.json")):
    sys.path.insert(0, REF_SRC)
    from infinisim import efficiency as E
    from infinisim import memory as M
    rows = []
    for s in SHAPES:
        cfg = M.ModelConfig(**s)
        row = {"shape": s,
               "params": M.param_count(cfg),
               "mswm_bytes": M.mswm_bytes(cfg),
               "awm_bytes": M.awm_bytes(cfg),
               "model_state_bytes": M.model_state_bytes(cfg),
               "flops_per_iter": float(E.compute_per_iter(cfg)),
               "ait": {k.value: E.ait(k, cfg) for k in E.AitKind}}
        rows.append(row)
    eff = []
    for a, bw, pk in itertools.product((1.0, 256.0, 1024.0, 49152.0, 196608.0), BWS, PEAKS):
        eff.append({"ait": a, "bw": bw if bw != float("inf") else "inf", "peak": pk,
                    "eff": E.efficiency(a, bw, pk)})
    req = [{"ait": a, "peak": pk, "target": t, "bw": E.required_bandwidth(a, pk, t)}
           for a, pk, t in itertools.product((1.0, 512.0, 49152.0), PEAKS, EFFS)]
    with open(out, "w") as f:
        json.dump({"source": "infinisim 0.1.0 memory.py / efficiency.py", "shapes": rows,
                   "efficiency": eff, "required_bandwidth": req,
                   "model_state_bytes_per_param": M.MODEL_STATE_BYTES_PER_PARAM}, f, indent=0)
    print(f"wrote {out}: {len(rows)} shapes, {len(eff)} efficiency, {len(req)} bandwidth points")


if __name__ == "__main__":
    main()
