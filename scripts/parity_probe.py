"""Measure the GPT engine's error against the CPU oracle (oracle/gpt.py), to set test tolerances.

Runs BASELINE config 1 (nl4 / hd256 / 4 heads / seq128 / batch4 / V512) at world 2 for
3 steps in bf16 and fp32 compute, and one step of a 1.3B-shape block (nl1, hd2048,
16 heads, seq1024, V50304, one sequence). Prints, per step: loss relative error,
per-bucket gradient-shard relative L2 (max over buckets), and the Adam update error
|dp_gpu - dp_oracle| in units of lr (max and 99.9th percentile) with the relative L2
of the update. Usage: python scripts/parity_probe.py [--act-ckpt host]
"""

import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import gpt as og  # noqa: E402
from oracle import numerics as nx  # noqa: E402
from paper_2104_07857_b200 import gpt as eg  # noqa: E402
from paper_2104_07857_b200.comm import LocalComm  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def run(cfg, world, steps, lr, compute, half_kind, act_ckpt=None, **kw):
    half = torch.bfloat16 if half_kind == nx.HALF_BF16 else torch.float16
    eng = eg.GPTZeroEngine(cfg, LocalComm(world), lr=lr, half_dtype=half, compute_dtype=compute,
                           act_ckpt=act_ckpt, **kw)
    eng.capture_grads = True
    oc = og.GPTConfig(cfg.nl, cfg.hd, cfg.heads, cfg.seq, cfg.vocab, cfg.batch)
    st = og.init_partitioned(oc, world, half_kind=half_kind)
    out = []
    for step in range(steps):
        prev = {k: [s.copy() for s in st.p32[k]] for k in st.p32}
        bs = [eg.synthetic_tokens(cfg, 7, r, step) for r in range(world)]
        t0 = time.time()
        loss = eng.step(bs).item()
        oloss, gsh = og.train_step(st, [(t.cpu().numpy(), y.cpu().numpy()) for t, y in bs], lr=lr)
        to = time.time() - t0
        g_rel = max(rel(eng.grad_shards[k][r].cpu().numpy(), gsh[k][r])
                    for k in gsh for r in range(world))
        g_worst = max(((k, r) for k in gsh for r in range(world)),
                      key=lambda kr: rel(eng.grad_shards[kr[0]][kr[1]].cpu().numpy(), gsh[kr[0]][kr[1]]))
        dmax, d999, urel, frac = 0.0, 0.0, 0.0, 0.0
        errs, nums, dens = [], 0.0, 0.0
        for k in st.p32:
            for r in range(world):
                p = eng.shard(k, r)["p32"].cpu().numpy().astype(np.float64)
                dg = p - prev[k][r]
                do = st.p32[k][r].astype(np.float64) - prev[k][r]
                e = np.abs(dg - do) / lr
                errs.append(e)
                nums += float(((dg - do) ** 2).sum())
                dens += float((do ** 2).sum())
        e = np.concatenate(errs)
        out.append({"step": step, "loss": loss, "oracle_loss": oloss,
                    "loss_rel": abs(loss - oloss) / abs(oloss), "grad_rel_max": g_rel,
                    "grad_worst": list(g_worst), "upd_err_max_lr": float(e.max()),
                    "upd_err_p999_lr": float(np.quantile(e, 0.999)),
                    "upd_err_frac_gt_0.1lr": float((e > 0.1).mean()),
                    "upd_err_frac_gt_1lr": float((e > 1.0).mean()),
                    "upd_rel_l2": float(np.sqrt(nums / max(dens, 1e-300))), "sec": round(to, 1)})
        print(json.dumps(out[-1]), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-big", action="store_true")
    args = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = False
    tiny = eg.TINY
    res = {}
    print("== config 1, bf16, world 2")
    res["c1_bf16"] = run(tiny, 2, 3, 1e-3, None, nx.HALF_BF16)
    print("== config 1, bf16, world 2, act_ckpt host")
    res["c1_bf16_ckpt"] = run(tiny, 2, 3, 1e-3, None, nx.HALF_BF16, act_ckpt="host")
    print("== config 1, fp32 compute, fp16 params, world 2")
    res["c1_fp32"] = run(tiny, 2, 3, 1e-3, torch.float32, nx.HALF_FP16)
    print("== config 1, bf16, world 2, cublas")
    res["c1_bf16_cublas"] = run(tiny, 2, 3, 1e-3, None, nx.HALF_BF16, gemm_select="cublas")
    print("== config 1, bf16, world 2, zi")
    res["c1_bf16_zi"] = run(tiny, 2, 3, 1e-3, None, nx.HALF_BF16, gemm_select="zi")
    if not args.skip_big:
        big = eg.GPTConfig(nl=1, hd=2048, heads=16, seq=1024, vocab=50304, batch=1)
        print("== 1.3B shape nl1, bf16, world 1")
        res["b_bf16"] = run(big, 1, 1, 1e-4, None, nx.HALF_BF16)
    with open("gpurun_out/parity_probe.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
