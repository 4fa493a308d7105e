"""Kernel-level timeline of graphed GPT-1.3B steps (torch.profiler / CUPTI): busy time per
stream, the union of busy intervals across streams, and the idle gaps inside the step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2104_07857_b200 import gpt as eg  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402

cfg = eg.GPT_1P3B
eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4)
bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
for s in range(4):
    eng.step_graphed([bs[s % 2]])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for s in range(2):
        eng.step_graphed([bs[s % 2]])
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev if e.time_range.end > e.time_range.start)
t0, t1 = iv[0][0], max(e for _, e, _ in iv)
union, cur_s, cur_e = 0.0, None, None
gaps, where = [], []
prev_name = None
for s, e, n in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            union += cur_e - cur_s
            gaps.append(s - cur_e)
            where.append((s - cur_e, prev_name, n, s - t0))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
    if e >= cur_e:
        prev_name = n
union += cur_e - cur_s
tot = sum(e - s for s, e, _ in iv)
by = {}
for s, e, n in iv:
    k = n[:60]
    by[k] = by.get(k, 0) + (e - s)
top = sorted(by.items(), key=lambda x: -x[1])[:25]
print(json.dumps({"span_ms": round((t1 - t0) / 1e3 / 2, 3), "busy_union_ms": round(union / 1e3 / 2, 3),
                  "kernel_sum_ms": round(tot / 1e3 / 2, 3), "n_gaps": len(gaps),
                  "gap_total_ms": round(sum(gaps) / 1e3 / 2, 3),
                  "gaps_over_5us": sum(1 for g in gaps if g > 5) // 2}))
for k, v in top:
    print(f"{v / 1e3 / 2:8.3f} ms  {k}")
for g, a, b, at in sorted(where, key=lambda w: -w[0])[:6]:
    print(f"gap {g:8.1f} us at {at / 1e3:8.3f} ms: after {str(a)[:50]} | before {str(b)[:50]}")
