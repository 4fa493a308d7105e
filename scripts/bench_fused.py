"""HBM roofline of the step's libzinf elementwise / reduction kernels at GPT-1.3B shapes.

One JSON line per kernel: warm average over `reps` launches (CUDA events), algorithmic
bytes per launch, GB/s and the fraction of MEASURED_PEAKS.json's HBM copy peak. The
operand set of each launch is cycled over several copies so consecutive launches do not
hit in L2.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_07857_b200 import kernels  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    PEAK = 6650.0
T, H, V = 8192, 2048, 50304
bf = torch.bfloat16


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


def report(name, ms, nbytes):
    gbs = nbytes / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": name, "us": round(ms * 1e3, 1), "mb": round(nbytes / 1e6, 1),
                      "gbs": round(gbs, 1), "frac": round(gbs / PEAK, 3)}), flush=True)


def main():
    ws = kernels.Workspace(max(4 << 20, 600 * 4 * H))
    C = 3   # operand copies cycled
    # LayerNorm forward with fused residual: read x, resid; write xsum, y (+ stats)
    xs = [torch.randn(T, H, device="cuda").to(bf) for _ in range(C)]
    rs = [torch.randn(T, H, device="cuda").to(bf) for _ in range(C)]
    w, bb = torch.ones(H, device="cuda", dtype=bf), torch.zeros(H, device="cuda", dtype=bf)
    ys = [torch.empty(T, H, device="cuda", dtype=bf) for _ in range(C)]
    ss = [torch.empty(T, H, device="cuda", dtype=bf) for _ in range(C)]
    mean = torch.empty(T, device="cuda")
    rstd = torch.empty(T, device="cuda")
    fns = [lambda i=i: kernels.ln_fwd(xs[i], w, bb, ys[i], mean, rstd, resid=rs[i], xsum=ss[i])
           for i in range(C)]
    report("ln_fwd+resid", timeit(fns), 4 * T * H * 2)
    fns = [lambda i=i: kernels.ln_fwd(xs[i], w, bb, ys[i], mean, rstd) for i in range(C)]
    report("ln_fwd", timeit(fns), 2 * T * H * 2)
    # LayerNorm backward with residual grad + dres column sum
    dws = torch.empty(H, device="cuda", dtype=bf)
    dbs = torch.empty(H, device="cuda", dtype=bf)
    drs = torch.empty(H, device="cuda", dtype=bf)
    fns = [lambda i=i: kernels.ln_bwd(ys[i], xs[i], w, mean, rstd, ss[i], dws, dbs, ws,
                                      dres=rs[i], dres_sum=drs) for i in range(C)]
    report("ln_bwd+dres", timeit(fns), 4 * T * H * 2)
    del xs, rs, ys, ss
    # GELU forward (fc1 activation): read u, write a (T x 4H)
    us = [torch.randn(T, 4 * H, device="cuda").to(bf) for _ in range(C)]
    As = [torch.empty(T, 4 * H, device="cuda", dtype=bf) for _ in range(C)]
    fns = [lambda i=i: kernels.gelu_fwd(us[i], As[i]) for i in range(C)]
    report("gelu_fwd", timeit(fns), 2 * T * 4 * H * 2)
    # GELU backward + fc1 bias grad: read da, u; write du; column sums
    db = torch.empty(4 * H, device="cuda", dtype=bf)
    fns = [lambda i=i: kernels.bias_grad(As[i], db, ws, u=us[i], du=As[(i + 1) % C])
           for i in range(C)]
    report("bias_grad+gelu_bwd", timeit(fns), 3 * T * 4 * H * 2)
    qs = [u.view(-1)[:T * 3 * H].view(T, 3 * H) for u in us]
    fns = [lambda i=i: kernels.bias_grad(qs[i], db[:3 * H], ws) for i in range(C)]
    report("bias_grad(qkv)", timeit(fns), T * 3 * H * 2)
    del us, As
    # softmax cross-entropy over the logits, in place: read + write T x V bf16
    lg = [torch.randn(T, V, device="cuda").to(bf) for _ in range(2)]
    tg = torch.randint(0, V, (T,), device="cuda")
    rows = torch.empty(T, device="cuda")
    loss = torch.empty((), device="cuda")
    fns = [lambda i=i: kernels.softmax_ce(lg[i], tg, rows, loss, 1.0 / T) for i in range(2)]
    report("softmax_ce", timeit(fns, 10), 2 * T * V * 2)


if __name__ == "__main__":
    main()
