"""zi_rs_adam_dc / zi_adam_step HBM throughput on a 1.3B block bucket (50.4M elements),
operands cycled over copies so launches do not hit in L2. One JSON line per variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import _lib, kernels  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
n = 50_358_272
C = 2
st = kernels.DeviceAdamState(1e-4, (0.9, 0.999), 1e-8)
st.advance()
sets = []
for _ in range(C):
    p = torch.rand(n, device="cuda") * 0.1
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    h = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    g = (torch.randn(n, device="cuda") * 1e-2).bfloat16()
    sets.append((p, m, v, h, g))


def t(fn, reps=20):
    for i in range(C):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps):
        fn(i % C)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


ms = t(lambda i: kernels.rs_adam_dc([sets[i][4]], 0, n, n, 1.0, *sets[i][:4], st))
gbs = 28 * n / ms / 1e6
print(json.dumps({"kernel": "zi_rs_adam_dc K=1", "us": round(ms * 1e3, 1), "gbs": round(gbs, 1),
                  "frac": round(gbs / PEAK, 4)}))
gs = [torch.randn(n, device="cuda") * 1e-2 for _ in range(C)]
cc = _lib.adam_consts(1e-4, 0.9, 0.999, 1e-8, 1)
ms = t(lambda i: kernels.adam_step(*sets[i][:3], gs[i], sets[i][3], cc))
gbs = 30 * n / ms / 1e6
print(json.dumps({"kernel": "zi_adam_step", "us": round(ms * 1e3, 1), "gbs": round(gbs, 1),
                  "frac": round(gbs / PEAK, 4)}))
a = torch.empty(n * 7, dtype=torch.float32, device="cuda")
bb = torch.empty_like(a)
ms = t(lambda i: bb.copy_(a))
print(json.dumps({"kernel": "torch copy (same bytes scale)", "gbs": round(2 * a.numel() * 4 / ms / 1e6, 1)}))
