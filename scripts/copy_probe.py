"""HBM copy bandwidth vs size (torch D2D copy_ and a plain vectorised copy kernel), timed
like scripts/bench_fused.py (warm, operand copies cycled so launches miss in L2)."""
import json
import torch

def timeit(fns, reps=30):
    for f in fns:
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps):
        fns[i % len(fns)]()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

for mb in (32, 64, 128, 512, 2048):
    n = mb << 20
    src = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(3)]
    dst = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(3)]
    ms = timeit([lambda i=i: dst[i].copy_(src[i]) for i in range(3)])
    print(json.dumps({"copy_mb": mb, "us": round(ms * 1e3, 1), "gbs": round(2 * n / ms / 1e6, 1)}))
