"""Sustained (power-capped) GEMM throughput and SM clock: each candidate loops one GEMM
for ~3 s while nvidia-smi samples clocks/power. python scripts/gemm_sustained.py [M N K]"""
import json, os, subprocess, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_07857_b200 import kernels  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (8192, 8192, 2048)
bf = torch.bfloat16
a = torch.randn(M, K, device="cuda", dtype=bf)
b = torch.randn(N, K, device="cuda", dtype=bf) * K ** -0.5
y = torch.empty(M, N, device="cuda", dtype=bf)
cands = {"zi_sk": lambda: kernels.gemm_sk(a, b, y), "zi_whole": lambda: kernels.gemm_sk(a, b, y, split=False),
         "cublas": lambda: torch.mm(a, b.t(), out=y)}
for name, fn in list(cands.items()) * 2:
    fn(); torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    e0.record()
    t0 = time.time()
    while time.time() - t0 < 3.0:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    vals = [tuple(float(x) for x in l.split(",")) for l in out[5:] if l.count(",") == 1]
    clk = sorted(v[0] for v in vals)[len(vals) // 2] if vals else None
    pw = sorted(v[1] for v in vals)[len(vals) // 2] if vals else None
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "tflops": round(2 * M * N * K / ms / 1e9, 1),
                      "sm_mhz": clk, "power_w": pw}), flush=True)
