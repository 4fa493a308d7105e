"""Benchmark: ZeRO-3 partitioned GPT training step on B200 (BASELINE config 2).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

* ``value``: whole-job model TFLOPS of the training step with inputs already
  resident in HBM, timed with CUDA events over exactly K steps (barrier +
  synchronize on both sides, max over ranks). TFLOPS/GPU = value / N; the
  line also carries samples/s.
* ``e2e``: the same metric through the public API (GPTZeroEngine.step) with
  the step's token batch copied from pinned host memory and the loss read
  back to the host every step.
* ``roofline``: the dominant kernel of the step, zi_gemm_sk (every linear,
  tensor-bound): sum of 2*M*N*K over its launches / sum of their CUDA-event
  durations inside a re-captured step, against the sustained bf16 peak.
  ``roofline_hbm``: the largest HBM-bound kernel (zi_rs_adam_dc, the fused
  reduce-scatter + Adam); per-launch duration measured with CUDA events on its
  stream inside the timed region.
* ``cpu_baseline`` / ``--impl reference``: the numpy oracle of the same step
  (oracle/gpt.py) on a bounded sample — one transformer block + embedding +
  head of the 1.3B shape, one 1024-token sequence — on the host cores.

Inputs: the step's working set (2.6 GB bf16 params, 15.8 GB fp32 optimizer
state, ~13 GB activations) is >100x the 126 MB L2, so no L2 flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

METRIC = "train TFLOPS/GPU + samples/s at 1/2/4/8 B200; all-gather/RS bus GB/s; offload GB/s"
ROOT = os.path.dirname(os.path.abspath(__file__))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback"


def _ncu_traffic(kernel: str, key: str = "dram_bytes_per_launch"):
    """DRAM read+write bytes per launch of ``kernel`` from the committed ncu --set full
    capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)[kernel][key]
    except Exception:  # noqa: BLE001
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        import threading
        self.lines = []
        first = threading.Event()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
            return self

        def read():
            for line in self.proc.stdout:
                self.lines.append(line)
                first.set()

        self.reader = threading.Thread(target=read, daemon=True)
        self.reader.start()
        # nvidia-smi takes a few hundred ms to start on some boxes: the timed region
        # begins only once it is sampling
        first.wait(timeout=5.0)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.reader.join(timeout=5)
            self.out = "".join(self.lines)
        return False

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                try:
                    rows.append((float(f[1]), float(f[2]), f[5:9]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = sorted(r[0] for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ CPU side
def cpu_sample(steps: int = 1):
    """The oracle (numpy) step on a bounded sample of the 1.3B workload.

    Returns (model TFLOPS, seconds per sample step, description, threads).
    """
    import numpy as np
    from oracle import gpt as og
    c = og.GPTConfig(nl=1, hd=2048, heads=16, seq=1024, vocab=50304, batch=1)
    st = og.init_partitioned(c, 1)
    flops = 6.0 * c.batch * c.seq * og.param_count(c) + 6 * 2 * c.batch * c.seq * c.seq * c.hd * c.nl
    times = []
    for s in range(steps):
        tok, tgt = og.synthetic_tokens(c, 7, 0, s)
        t0 = time.perf_counter()
        og.train_step(st, [(tok, tgt)], lr=1e-4)
        times.append(time.perf_counter() - t0)
    dt = min(times)
    desc = ("numpy oracle train_step (oracle/gpt.py): 1 block + tied embedding/head of the 1.3B "
            "shape (hd 2048, V 50304), 1 x 1024 tokens, fwd+bwd+RS+Adam")
    return flops / dt / 1e12, dt, desc, len(os.sched_getaffinity(0))


def cpu_components() -> dict:
    """SURVEY §8(d)'s per-path CPU baselines on the host cores, each a bounded sample:
    the reference tier store itself (baseline/_ref, unmodified) host- and NVMe-tier
    write/read GB/s, and the numpy oracle's Adam, reduce-scatter and tiled linear."""
    import tempfile
    import numpy as np
    from oracle import numerics as nx
    from oracle.adam import AdamConsts, adam_update
    from oracle.partition import reduce_scatter_cast
    from oracle.tiling import forward_tiled
    out = {}

    def best(fn, reps=3):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    # reference store (pkg/src/infinisim/store.py) through its own public API
    ref = os.path.join(ROOT, "baseline", "_ref")
    try:
        sys.path.insert(0, ref)
        from infinisim import store as R  # noqa: E402
        a = np.random.default_rng(0).standard_normal(32 << 20).astype(np.float32)  # 128 MiB
        nb = a.nbytes
        with tempfile.TemporaryDirectory() as d:
            st = R.TierStore(0, 4 * nb, nvme_root=d, nvme_capacity=4 * nb)
            for tier, name in ((R.TierKind.HOST, "host"), (R.TierKind.NVME, "nvme")):
                tw = best(lambda: st.flush([st.write("x", a, tier)]))
                tr = best(lambda: st.read("x", tier).wait())
                out[f"reference_store_{name}_write_gbs"] = round(nb / tw / 1e9, 2)
                out[f"reference_store_{name}_read_gbs"] = round(nb / tr / 1e9, 2)
                st.delete("x", tier)
            st.close()
        out["reference_store_sample"] = "128 MiB f32 array, best of 3 (NVMe tier: OS page cache)"
    except Exception as e:  # noqa: BLE001
        out["reference_store"] = f"unavailable: {e!r}"[:200]
    finally:
        if sys.path and sys.path[0] == ref:
            sys.path.pop(0)
    rng = np.random.default_rng(1)
    n = 16 << 20
    p, m, g = (rng.standard_normal(n).astype(np.float32) for _ in range(3))
    v = np.abs(rng.standard_normal(n)).astype(np.float32)
    c = AdamConsts.make(1e-4, 0.9, 0.999, 1e-8, 3)
    t = best(lambda: adam_update(p, m, v, g, c))
    out["oracle_adam_gbs"] = round(n * 30 / t / 1e9, 2)
    out["oracle_adam_melem_s"] = round(n / t / 1e6, 1)
    world, n = 8, 4 << 20
    cs = [nx.half_bits_to_f32(nx.f32_to_half_bits(rng.standard_normal(n).astype(np.float32),
                                                  nx.HALF_BF16), nx.HALF_BF16)
          for _ in range(world)]
    t = best(lambda: reduce_scatter_cast(cs, world, 1.0 / world))
    out["oracle_reduce_scatter_gbs"] = round(world * n * 2 / t / 1e9, 2)
    W = rng.standard_normal((4096, 4096)).astype(np.float32)
    b = rng.standard_normal(4096).astype(np.float32)
    x = rng.standard_normal((1024, 4096)).astype(np.float32)
    t = best(lambda: forward_tiled(W, b, x, 4))
    out["oracle_tiled_linear_gflops"] = round(2 * 1024 * 4096 * 4096 / t / 1e9, 1)
    out["components_sample"] = ("Adam 16M fp32 elems (30 B/elem); RS 8 ranks x 4M bf16 "
                                "(bus bytes = 8*n*2); tiled linear M=1024, 4096->4096, T=4 fp32")
    return out


def tiling_leg(T: int = 8, iters: int = 5) -> dict:
    """BASELINE config 4 at one tile count: the 16384 -> 65536 linear over M = 8192 tokens
    split into T row tiles, forward_tiled / backward_tiled through the tier store (each
    tile fetched just in time into a 2-slot ring), every tile product on tcgen05
    (zi_linear_tile_fwd / _bwd). The roofline is the tile kernel timed alone (CUDA events)
    against the burst bf16 peak; cuBLAS on the same tiles beside it."""
    import tempfile
    import torch
    from paper_2104_07857_b200 import kernels
    from paper_2104_07857_b200.store import TierKind, TierStore
    from paper_2104_07857_b200.tiling import backward_tiled, forward_tiled, tile_linear
    M, K, N = 8192, 16384, 65536
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16, generator=g)
    W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16, generator=g) * K ** -0.5
    b = torch.randn(N, device="cuda", dtype=torch.bfloat16, generator=g)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gy = (torch.randn(M, N, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)

    def timed(fn, n=iters):
        fn()
        torch.cuda.synchronize()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        c.record()
        torch.cuda.synchronize()
        return a.elapsed_time(c) / n

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        burst = json.load(f)["bf16_tflops"]
    out = {"workload": f"tiled linear 16384->65536, T={T}, M={M} tokens, bf16"}
    with TierStore(16 << 30, 1 << 30, nvme_root=tempfile.mkdtemp()) as st:
        tl = tile_linear(W, b, T, st, TierKind.DEVICE, key="c4")
        ms_f = timed(lambda: forward_tiled(tl, x, st, out=y))
        ms_b = timed(lambda: backward_tiled(tl, x, gy, st), max(2, iters // 2))
    s0, e0 = 0, N // T

    def cub():
        for s, e in ((i * (N // T), (i + 1) * (N // T)) for i in range(T)):
            torch.addmm(b[s:e], x, W[s:e].t(), out=y[:, s:e]) if y[:, s:e].is_contiguous() \
                else y[:, s:e].copy_(torch.addmm(b[s:e], x, W[s:e].t()))
    ms_c = timed(cub)
    Wt, yt = W[s0:e0], torch.empty(M, e0 - s0, device="cuda", dtype=torch.bfloat16)
    ms_k = timed(lambda: kernels.linear_fwd(x, Wt, b[s0:e0], yt))
    tf_k = 2.0 * M * K * (e0 - s0) / (ms_k / 1e3) / 1e12
    out.update({"forward_tiled_ms": round(ms_f, 3),
                "forward_tflops": round(2.0 * M * K * N / (ms_f / 1e3) / 1e12, 1),
                "backward_tiled_ms": round(ms_b, 3),
                "backward_tflops": round(4.0 * M * K * N / (ms_b / 1e3) / 1e12, 1),
                "cublas_same_tiles_fwd_ms": round(ms_c, 3),
                "roofline": {"kernel": "zi_linear_tile_fwd (2-SM tcgen05, one tile alone)",
                             "bound": "tensor", "achieved": round(tf_k, 1), "peak": burst,
                             "peak_kind": "measured burst", "unit": "TFLOP/s",
                             "frac": round(tf_k / burst, 4),
                             "ncu": "profiles/r1_gemm_tile_ncu.md (tensor pipe 98.0 % active)"}})
    del x, W, y, gy
    torch.cuda.empty_cache()
    return out


def store_leg() -> dict:
    """The tier store through the reference API on the GPU box, on
    the same 128 MiB f32 sample as cpu_components' reference-store numbers: HOST tier
    (pinned DRAM) and NVME tier (.shard files via the native pinned pool) from a numpy
    array, DEVICE tier (HBM) from a CUDA tensor. Host wall clock, best of 3."""
    import tempfile
    import numpy as np
    import torch
    from paper_2104_07857_b200 import store as S
    a = np.random.default_rng(0).standard_normal(32 << 20).astype(np.float32)
    nb = a.nbytes
    out = {}

    def best(fn, reps=3):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    with tempfile.TemporaryDirectory() as d:
        with S.TierStore(4 * nb, 4 * nb, nvme_root=d, nvme_capacity=4 * nb) as st:
            src = {S.TierKind.HOST: a, S.TierKind.NVME: a,
                   S.TierKind.DEVICE: torch.from_numpy(a).cuda()}
            for tier, name in ((S.TierKind.DEVICE, "device"), (S.TierKind.HOST, "host"),
                               (S.TierKind.NVME, "nvme")):
                def rd():
                    st.read("x", tier).wait()
                    torch.cuda.synchronize()
                tw = best(lambda: (st.flush([st.write("x", src[tier], tier)]),
                                   torch.cuda.synchronize()))
                tr = best(rd)
                out[f"{name}_write_gbs"] = round(nb / tw / 1e9, 2)
                out[f"{name}_read_gbs"] = round(nb / tr / 1e9, 2)
                st.delete("x", tier)
    out["sample"] = "128 MiB f32 array, best of 3, host wall clock; NVMe tier: OS page cache"
    return out


def run_reference(args):
    """--impl reference: the CPU oracle of the path on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(v, str(threads))
    cpu_sample(max(1, min(args.warmup, 1)))  # warm-up (numpy/BLAS init)
    tf, dt, desc, cores = cpu_sample(max(1, args.steps))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(tf, 6), "unit": "TFLOPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": "GPT-1.3B ZeRO-3 step (bounded CPU sample)", "global_batch": 1,
                   "seq_len": 1024, "parallelism": "cpu"},
        "cpu_baseline": {"value": round(tf, 6), "unit": "TFLOPS", "cores": cores, "kind": "port",
                         "sample": desc},
        "e2e": {"value": round(tf, 6), "unit": "TFLOPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU side
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2104_07857_b200 import gpt as eg
    from paper_2104_07857_b200.comm import DistComm, LocalComm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # ZINF_BENCH_SAME_GPU=1 (tests only): every rank on cuda:0 with gloo as the
    # process-group backend, to exercise the multi-process path on one GPU
    same_gpu = os.environ.get("ZINF_BENCH_SAME_GPU") == "1"
    torch.cuda.set_device(0 if same_gpu else local)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = DistComm()
    else:
        comm = LocalComm(1)
    cfg = eg.GPT_1P3B
    eng = eg.GPTZeroEngine(cfg, comm, seed=7, lr=1e-4)
    from paper_2104_07857_b200 import gemm_select
    # every site runs on zi_gemm_sk; the comparison column times cuBLAS on the same
    # shapes (outside the timed region), so the line shows what the library would do
    gemm_sites = gemm_select.compare_gpt(cfg.batch * cfg.seq, cfg.hd, cfg.vocab, eng.ws, eng.dev)
    for v in gemm_sites.values():
        v["faster"] = v.pop("choice")
        v["runs"] = "zi_gemm_sk" if eng.gemm_select == "zi" else eng.gemm_select

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # device-resident synthetic batches (distinct per step)
    dev_batches = [eg.synthetic_tokens(cfg, 7, rank, s) for s in range(max(args.steps, 1))]

    # ---------------- kernel-level roofline instrumentation: CUDA events around every
    # zi_rs_adam launch on its stream. Under CUDA graphs the events are captured
    # into the graph, so each replay re-times the launches of that step.
    from paper_2104_07857_b200 import kernels as K
    orig = K.rs_adam_dc
    rec = []

    def timed_rs_adam(*a, **kw):
        tm = K.GraphTimer()      # external event records: re-timed on every graph replay
        tm.start()
        orig(*a, **kw)
        tm.stop()
        n = a[2]
        ncontrib = len(a[0])
        rec.append((tm, None, n * (2 * ncontrib + 12 + 14), torch.cuda.is_current_stream_capturing()))

    K.rs_adam_dc = timed_rs_adam
    # multi-process too: the zi_ctx barriers take their epochs from device counters, so
    # the captured step (P2P gathers, barriers, RS + Adam over peer buckets) replays
    step = eng.step if args.no_graph else eng.step_graphed
    for w in range(args.warmup):
        step([dev_batches[w % len(dev_batches)]])
    barrier()
    if args.no_graph:
        rec.clear()

    # ---------------- timed region (device-resident inputs)
    launches0 = eng.launches
    clocks = ClockSampler(local)
    with clocks:
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for s in range(args.steps):
            loss = step([dev_batches[s % len(dev_batches)]])
        t1.record()
        barrier()
    K.rs_adam_dc = orig
    rec = [r for r in rec if r[3]] if not args.no_graph else rec
    ms = t0.elapsed_time(t1)
    if world > 1:
        ms = comm.allreduce_max(ms)
    launches = eng.launches - launches0
    ms_step = ms / args.steps
    flops = eg.model_flops_per_step(cfg)          # per rank
    tflops_job = flops * world / (ms_step / 1e3) / 1e12
    samples_s = cfg.batch * world / (ms_step / 1e3)
    k_ms = [tm.ms() for tm, _, _, _ in rec]
    k_bytes = [nb for _, _, nb, _ in rec]
    hbm, tc, peak_kind = _peaks()
    # the largest bucket's launches (the 24 block buckets) dominate
    # the transformer-block buckets (24 of the 26 launches per step) dominate
    big = max(set(k_bytes), key=k_bytes.count) if k_bytes else 0
    sel = [(t, b) for t, b in zip(k_ms, k_bytes) if b == big]
    avg_ms = sum(t for t, _ in sel) / max(1, len(sel))
    achieved = big / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else 0.0
    per_step = sum(k_ms) if not args.no_graph else sum(k_ms) / args.steps
    rs_share = per_step / ms_step if ms_step > 0 else 0.0

    # ---------------- e2e through the public API with host buffers
    import numpy as np
    host = []
    for s in range(args.steps):
        tok = torch.from_numpy(np.random.default_rng([7, rank, 1000 + s]).integers(
            0, cfg.vocab, size=(cfg.batch, cfg.seq + 1), dtype=np.int64)).pin_memory()
        host.append(tok)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(args.steps):
        d = host[s].to("cuda", non_blocking=True)
        loss = step([(d[:, :-1], d[:, 1:])])
        _ = loss.item()
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        e2e_ms = comm.allreduce_max(e2e_ms)
    e2e_tflops = flops * world / (e2e_ms / args.steps / 1e3) / 1e12

    # ---------------- tensor roofline of the dominant kernel (zi_gemm_sk: every linear of
    # the step). Separate from the headline: the step is re-captured with CUDA events
    # around each GEMM launch (event nodes cost the GEMMs their PDL overlap, so this
    # under-states them slightly), replayed `gsteps` times; 2*M*N*K flops per launch.
    # N=1 only: the re-capture runs host barriers across ranks, and an error on one rank
    # inside it would leave the others waiting; at N>1 `roofline` is the RS + Adam kernel.
    gemm_roof = None
    if not args.no_graph and world == 1:
        try:
            gemm_roof = gemm_roofline(eng, step, dev_batches, tc, min(args.steps, 5))
        except Exception as e:  # noqa: BLE001 — report, never lose the main line
            gemm_roof = {"error": repr(e)[:300]}

    # ---------------- collectives over NVLink (N > 1): bus GB/s of the step's AG / RS;
    # at N=1 the same kernels over 8 simulated ranks' buffers in this GPU's HBM
    collectives = None
    if world == 1:
        try:
            collectives = local_collective_kernels(eng)
        except Exception as e:  # noqa: BLE001 — report, never lose the main line
            collectives = {"error": repr(e)[:300]}
    if world > 1:
        try:
            collectives = collective_leg(eng, comm)
            if same_gpu:   # every rank time-shares one GPU: local HBM copies, not NVLink
                collectives["link"] = ("local HBM: ranks time-share one GPU (ZINF_BENCH_SAME_GPU); "
                                       "not an NVLink bus bandwidth")
                collectives.pop("nvlink_ref_gbs", None)
        except Exception as e:  # noqa: BLE001 — report, never lose the main line
            collectives = {"error": repr(e)[:300]}

    # ---------------- offload leg: fp32 optimizer state in pinned host DRAM
    offload = None
    config3_real = None
    if world == 1 and not args.no_offload:
        del eng
        torch.cuda.empty_cache()
        if not args.no_config3:   # first, while this process holds no pinned arenas
            config3_real = _leg_subprocess("config3_real", args)
        try:
            offload = offload_leg(cfg, args)
        except Exception as e:  # noqa: BLE001 — report, never lose the main line
            import traceback
            traceback.print_exc()
            offload = {"error": repr(e)[:300]}
            torch.cuda.synchronize()

    store = tiling = None
    if world == 1 and not args.no_offload:
        store = _safe(store_leg)
        tiling = _safe(tiling_leg)
        if offload is not None and config3_real is not None:
            offload["config3_real"] = config3_real

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        tf, dt, desc, cores = cpu_sample(1)
        cpu = {"value": round(tf, 6), "unit": "TFLOPS", "cores": cores, "kind": "port",
               "sample": desc, "sec_per_sample": round(dt, 3)}
        try:
            cpu["components"] = cpu_components()
        except Exception as e:  # noqa: BLE001 — report, never lose the main line
            cpu["components"] = {"error": repr(e)[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(tflops_job, 3), "unit": "TFLOPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "same_gpu": same_gpu, "physical_gpus": 1 if same_gpu else world,
            "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "GPT-style 1.3B (24 layers, hidden 2048, 16 heads, seq 1024, "
                                   "vocab 50304, tied) ZeRO-3 bf16, all states in HBM",
                       "global_batch": cfg.batch * world, "per_gpu_batch": cfg.batch,
                       "seq_len": cfg.seq, "parallelism": f"zero3-dp{world}",
                       "l2": "working set > 100x L2 (no flush needed)"},
            "tflops_per_gpu": round(tflops_job / world, 3),
            "samples_per_s": round(samples_s, 3),
            "flops_per_step_per_gpu": flops,
            "flops_formula": "6*tokens*params + 12*B*S^2*hd*nl (attention at the dense-equivalent "
                             "count, the MFU convention; no recompute)",
            "tflops_per_gpu_causal_executed": round(
                eg.model_flops_per_step(cfg, causal_executed=True) / (ms_step / 1e3) / 1e12, 3),
            "loss": float(loss.item()),
            "e2e": {"value": round(e2e_tflops, 3), "unit": "TFLOPS",
                    "h2d_bytes_per_step": cfg.batch * (cfg.seq + 1) * 8,
                    "d2h_bytes_per_step": 4},
            "gpu_launches": launches,
            "gemm_sites": gemm_sites,
            "roofline_hbm": {"kernel": "zi_rs_adam_dc (fused RS + cast + Adam over a block bucket's "
                                   "shard: 2 B per contribution + 26 B per shard element)",
                         "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4),
                         "bytes_per_launch": big, "avg_launch_ms": round(avg_ms, 4),
                         "share_of_step": round(rs_share, 4),
                         # the ncu capture is of the N=1 launch (50.4M elements, 1 contribution)
                         "traffic": _ncu_traffic("zi_rs_adam_dc") if world == 1 else None},
            "clocks": clocks.summary(),
            "offload": offload,
            "collectives": collectives,
            "store": store,
            "tiling": tiling,
            "cpu_baseline": cpu,
        }
        # `roofline` is the dominant kernel of the step: zi_gemm_sk (tensor-bound, ~70 % of
        # the step); the fused RS + Adam (the largest HBM-bound kernel) is `roofline_hbm`
        if gemm_roof is not None and "error" not in gemm_roof:
            line["roofline"] = gemm_roof
        else:
            line["roofline"] = line["roofline_hbm"]
            if gemm_roof is not None:
                line["roofline_gemm_error"] = gemm_roof
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def gemm_roofline(eng, step, batches, peak_tflops, gsteps: int) -> dict:
    """zi_gemm_sk inside the captured step: Σ 2·M·N·K over the step's GEMM launches ÷ Σ of
    their CUDA-event durations (external event records captured around each launch,
    re-timed on every replay), against the sustained bf16 peak (timed inside a long
    step)."""
    import torch
    from paper_2104_07857_b200 import kernels as K
    orig = K.gemm_sk
    rec = []

    def timed(a, b, out, *args, **kw):
        s = kw.get("stream")
        tm = K.GraphTimer()
        tm.start(s)
        r = orig(a, b, out, *args, **kw)
        tm.stop(s)
        nb = (a.numel() + b.numel()) * 2 + out.numel() * out.element_size()
        nb += sum(t.numel() * 2 for t in (kw.get("x"), kw.get("out2")) if t is not None)
        rec.append((tm, 2 * a.shape[0] * b.shape[0] * a.shape[1],
                    torch.cuda.is_current_stream_capturing(), nb))
        return r

    K.gemm_sk = timed
    try:
        eng._graph = None                     # re-capture with the timers in the graph
        step([batches[0]])
        rec[:] = [r for r in rec if r[2]]     # the captured launches only
        torch.cuda.synchronize()
        tot_ms, tot_fl = [], 0
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        step_ms = []
        for s in range(gsteps):
            t0.record()
            step([batches[s % len(batches)]])
            t1.record()
            torch.cuda.synchronize()
            step_ms.append(t0.elapsed_time(t1))
            tot_ms.append(sum(r[0].ms() for r in rec))
        tot_fl = sum(r[1] for r in rec)
        alg_b = sum(r[3] for r in rec)
    finally:
        K.gemm_sk = orig
        eng._graph = None
    g_ms = sorted(tot_ms)[len(tot_ms) // 2]
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            burst = json.load(f)["bf16_tflops"]
    except Exception:  # noqa: BLE001
        burst = None
    traffic = _ncu_traffic("zi_gemm_sk", "dram_bytes_per_step")
    st_ms = sorted(step_ms)[len(step_ms) // 2]
    achieved = tot_fl / (g_ms / 1e3) / 1e12
    return {"kernel": "zi_gemm_sk (stream-K tcgen05, CTA pairs; all %d GEMM launches of the "
                      "step: every linear fwd/dgrad/wgrad + the tied head)" % len(rec),
            "bound": "tensor", "achieved": round(achieved, 1), "peak": peak_tflops,
            "peak_kind": "measured sustained (kernel timed inside a long step)",
            "unit": "TFLOP/s", "frac": round(achieved / peak_tflops, 4),
            "flops_per_step": tot_fl, "launches_per_step": len(rec),
            "avg_launch_ms": round(g_ms / max(1, len(rec)), 4),
            "gemm_ms_per_step": round(g_ms, 3),
            "share_of_step": round(g_ms / st_ms, 4) if st_ms > 0 else None,
            "instrumented_step_ms": round(st_ms, 3),
            "frac_of_burst_peak": round(achieved / burst, 4) if burst else None,
            "algorithmic_bytes_per_step": alg_b,
            "traffic": traffic,
            "traffic_note": "ncu DRAM read+write per step (profiles/r2_gemm_step_ncu_s5.md) vs the "
                            "operand/output bytes: re-reads, but ~2 TB/s average, tensor-bound"}


def local_collective_kernels(eng, ranks: int = 8, iters: int = 10) -> dict:
    """N=1: the step's gather and reduce-scatter kernels over `ranks` simulated ranks' buffers
    of one 1.3B block bucket in this GPU's HBM (shards / gradient buckets at distinct
    addresses, as the IPC-mapped peers would be). Not NVLink numbers: HBM GB/s of the
    kernels themselves (gather: shard bytes read + full bytes written; RS: every rank's
    bf16 bucket read over our shard + the fp32 shard written), against the copy peak."""
    import torch
    from paper_2104_07857_b200 import kernels as K
    b = eng.by_key["h0"]
    n = b.numel
    L = -(-n // ranks)
    shards = [torch.randint(-3000, 3000, (L,), dtype=torch.int16, device="cuda").view(torch.bfloat16)
              for _ in range(ranks)]
    full = torch.empty(L * ranks, dtype=torch.bfloat16, device="cuda")
    grads = [torch.randn(n, device="cuda").bfloat16() for _ in range(ranks)]
    out = torch.empty(L, dtype=torch.float32, device="cuda")
    hbm, _, _ = _peaks()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    res = {"what": f"{ranks} simulated ranks in one GPU's HBM (not NVLink): kernel GB/s",
           "bucket_elems": n}
    ag_bytes = 2 * 2 * n
    for name, ce in (("allgather_sm", False), ("allgather_ce", True)):
        ms = timed(lambda: K.allgather(shards, L, full, n, use_copy_engine=ce))
        res[f"{name}_ms"] = round(ms, 4)
        res[f"{name}_gbs"] = round(ag_bytes / (ms / 1e3) / 1e9, 1)
    rs_bytes = ranks * 2 * L + 4 * L
    # one rank's shard of the rank-order fold (each rank runs this for its own shard)
    ms = timed(lambda: K.reduce_scatter_cast(grads, 3 * L, L, n, 1.0 / ranks, torch.bfloat16, out))
    res["reduce_scatter_ms"] = round(ms, 4)
    res["reduce_scatter_gbs"] = round(rs_bytes / (ms / 1e3) / 1e9, 1)
    res["reduce_scatter_frac_of_hbm_peak"] = round(rs_bytes / (ms / 1e3) / 1e9 / hbm, 4)
    res["allgather_sm_frac_of_hbm_peak"] = round(res["allgather_sm_gbs"] / hbm, 4)
    del shards, full, grads, out
    torch.cuda.empty_cache()
    return res


def collective_leg(eng, comm, iters: int = 10) -> dict:
    """Bus GB/s of the step's collectives on one block bucket (bf16, ~100 MB at 1.3B):
    the P2P all-gather (zi_allgather pulling every peer's shard over NVLink), the
    fused P2P reduce-scatter (zi_reduce_scatter_cast folding the peers' gradient
    buckets in rank order) and NCCL's all_gather_into_tensor for reference.
    bus bytes = S * (N-1) / N per rank (S = full bucket bytes); max time over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2104_07857_b200 import kernels as K
    N = comm.world
    b = eng.by_key["h0"]
    S = b.numel * 2
    full = torch.empty(b.shard * N, dtype=torch.bfloat16, device="cuda")
    shard32 = torch.empty(b.shard, dtype=torch.float32, device="cuda")
    p16_ptrs = [p + b.arena_off * 2 for p in eng.peer_p16] if hasattr(eng, "peer_p16") else None
    g_ptrs = list(eng.peer_gslots[0])
    out = {"bucket_bytes": S, "n_ranks": N}

    def timed(fn):
        comm.device_barrier(channel=3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return comm.allreduce_max(e0.elapsed_time(e1) / iters)

    def bus(ms):
        return round(S * (N - 1) / N / (ms / 1e3) / 1e9, 1)

    if p16_ptrs is not None:
        ms = timed(lambda: K.allgather(p16_ptrs, b.shard, full, b.numel))
        out["allgather_p2p_ms"], out["allgather_p2p_busbw_gbs"] = round(ms, 4), bus(ms)
        ms = timed(lambda: K.allgather(p16_ptrs, b.shard, full, b.numel, use_copy_engine=True))
        out["allgather_ce_ms"], out["allgather_ce_busbw_gbs"] = round(ms, 4), bus(ms)
    r = comm.rank
    ms = timed(lambda: K.reduce_scatter_cast(g_ptrs, r * b.shard, b.shard, b.numel, 1.0 / N,
                                             torch.bfloat16, shard32))
    out["reduce_scatter_p2p_ms"], out["reduce_scatter_p2p_busbw_gbs"] = round(ms, 4), bus(ms)
    if comm.backend == "nccl":
        mine = eng.p16[0, b.arena_off:b.arena_off + b.shard]
        ms = timed(lambda: dist.all_gather_into_tensor(full, mine))
        out["allgather_nccl_ms"], out["allgather_nccl_busbw_gbs"] = round(ms, 4), bus(ms)
    out["nvlink_ref_gbs"] = 770.0
    # bandwidth-centric partitioning A/B through the SPEC API: the
    # bucket as a PartitionedTensor gathered from every rank's shard vs the whole bucket
    # pulled from one owner (broadcast_fetch); effective GB/s = bucket bytes delivered
    # to each rank per second (allgather should scale with N, the broadcast stays flat)
    try:
        from paper_2104_07857_b200.partition import allgather, broadcast_fetch, partition
        from paper_2104_07857_b200.store import TierKind, TierStore
        import tempfile
        st = TierStore(4 * S + (64 << 20), 0, nvme_root=tempfile.mkdtemp(prefix="zinf-ab-"))
        src = torch.empty(b.numel, dtype=torch.bfloat16, device="cuda").normal_()
        pt = partition(src, N, TierKind.DEVICE, st, key="ab.bucket", comm=comm)
        if r == 0:
            st.write("ab.whole", src, TierKind.DEVICE).wait()
        ag_out = torch.empty(b.numel, dtype=torch.bfloat16, device="cuda")
        ms_ag = timed(lambda: allgather(pt, st, comm, out=ag_out, use_copy_engine=True))
        ms_bc = timed(lambda: broadcast_fetch("ab.whole", TierKind.DEVICE, st, comm=comm, owner=0,
                                              numel=b.numel, dtype=torch.bfloat16))
        out["spec_api_ab"] = {"allgather_ms": round(ms_ag, 4), "broadcast_fetch_ms": round(ms_bc, 4),
                              "allgather_eff_gbs": round(S / (ms_ag / 1e3) / 1e9, 1),
                              "broadcast_eff_gbs": round(S / (ms_bc / 1e3) / 1e9, 1)}
        st.close()
    except Exception as e:  # noqa: BLE001 — report, never lose the main line
        out["spec_api_ab"] = {"error": repr(e)[:300]}
    return out


def host_link_peak(nbytes: int = 1 << 30) -> dict:
    """Pinned cudaMemcpyAsync H2D, D2H and both at once (copy engines), GB/s."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d: bool, d2h: bool) -> float:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            if h2d:
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        return 3 * nbytes * (int(h2d) + int(d2h)) / (time.perf_counter() - t0) / 1e9
    run(True, True)
    return {"h2d_gbs": round(run(True, False), 1), "d2h_gbs": round(run(False, True), 1),
            "duplex_gbs": round(run(True, True), 1)}


def offload_leg(cfg, args) -> dict:
    """The 1.3B step with fp32 master/m/v in pinned host memory (ZeRO-Offload placement;
    per-GPU traffic equals BASELINE config 3's 10B/8 shard), streamed per bucket through
    the H2D || rs_adam || D2H pipeline during backward."""
    import torch
    from paper_2104_07857_b200 import gpt as eg
    from paper_2104_07857_b200.comm import LocalComm
    from paper_2104_07857_b200.store import TierKind
    peak = host_link_peak()
    eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4,
                           placement=eg.Placement(TierKind.DEVICE, TierKind.HOST))
    bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
    for w in range(2):
        eng.step([bs[w % 2]])
    torch.cuda.synchronize()
    b0 = eng.offload_bytes
    steps = max(2, min(args.steps, 5))
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in range(steps):
        eng.step([bs[s % 2]])
    eng.flush()          # the last step's deferred write-back is inside the timed region
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    moved = (eng.offload_bytes - b0) / steps
    eng.trace = True          # one extra traced step for the overlap Timeline
    eng.step([bs[0]])
    tl = eng.timeline()
    cal = {}
    for name, duplex in (("half_duplex", False), ("duplex", True)):
        sim = eng.simulated_step(duplex)
        cal["measured_step_s"] = round(sim["measured_s"], 4)
        cal[f"predicted_{name}_s"] = round(sim["predicted_s"], 4)
        cal[f"rel_error_{name}"] = round(sim["rel_error"], 4)
    eng.trace = False
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "offload_timeline.csv"), "w") as f:
        f.write(tl.to_csv())
    out = {"workload": "GPT-1.3B ZeRO-3 step, fp32 optimizer state (15.8 GB) in pinned host DRAM",
           "ms_per_step": round(ms, 2),
           "tflops": round(eg.model_flops_per_step(cfg) / (ms / 1e3) / 1e12, 1),
           "host_bytes_per_step": int(moved),
           "host_link_gbs": round(moved / (ms / 1e3) / 1e9, 1),
           "host_link_peak": peak,
           "frac_of_duplex_peak": round(moved / (ms / 1e3) / 1e9 / peak["duplex_gbs"], 3),
           "timeline": {"pcie_busy_s": round(tl.lane_busy_s("pcie"), 4),
                        "compute_busy_s": round(tl.lane_busy_s("compute"), 4),
                        "traced_step_s": round(tl.total_s, 4),
                        "pcie_hidden_behind_compute": round(tl.hidden_fraction(("pcie",)), 4)},
           "simulator_calibration": cal}
    del eng
    torch.cuda.empty_cache()
    # activation checkpoints offloaded to pinned host (PAPER §5.1.2): forward keeps each
    # block input (D2H), backward prefetches it one block ahead and recomputes the block
    eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4, act_ckpt="host")
    for w in range(2):
        eng.step_graphed([bs[w % 2]])
    torch.cuda.synchronize()
    t0.record()
    for s in range(steps):
        eng.step_graphed([bs[s % 2]])
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    eng.trace = True
    eng.step([bs[0]])
    tl = eng.timeline()
    sim = eng.simulated_step()
    T, P = cfg.tokens, eg.param_count(cfg)
    out["act_ckpt_host"] = {
        "ms_per_step": round(ms, 2),
        "model_tflops": round(eg.model_flops_per_step(cfg) / (ms / 1e3) / 1e12, 1),
        "hw_tflops_8TP": round((8.0 * T * P + 8 * 2 * cfg.batch * cfg.seq ** 2 * cfg.hd * cfg.nl)
                               / (ms / 1e3) / 1e12, 1),
        "ckpt_bytes_per_step": 2 * cfg.nl * T * cfg.hd * 2,
        "pcie_hidden_behind_compute": round(tl.hidden_fraction(("pcie",)), 4),
        "simulator_calibration": {"measured_step_s": round(sim["measured_s"], 4),
                                  "predicted_s": round(sim["predicted_s"], 4),
                                  "rel_error": round(sim["rel_error"], 4)}}
    del eng
    torch.cuda.empty_cache()
    out["config3_equiv"] = _safe(offload_equiv_leg, args)
    out["config5_equiv"] = _safe(offload_equiv_leg, args, batch=32, params_host=True)
    if not args.no_nvme:
        out["nvme_params"] = _safe(nvme_params_leg, cfg, args, bs, steps)
        out["nvme_optimizer"] = _safe(nvme_leg, cfg, args, bs, steps)
        out["nvme_optimizer_direct"] = _safe(nvme_leg, cfg, args, bs, 1, direct=True)
    return out


def _safe(fn, *a, **kw) -> dict:
    """Run one bench sub-leg; a failure is reported in its slot, never loses the line."""
    import gc
    import torch
    try:
        return fn(*a, **kw)
    except Exception as e:  # noqa: BLE001
        import traceback
        traceback.print_exc()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        return {"error": repr(e)[:300]}
    finally:
        gc.collect()     # free the leg's engines (and their pinned arenas) now


def offload_equiv_leg(args, batch: int = 64, params_host: bool = False) -> dict:
    """A BASELINE config's per-GPU balance on one GPU: 1.3B with ``batch`` sequences.

    Config 3 (10B, N=8): each GPU has 8*8192*10.28e9 = 6.7e14 step flops and a 1.28 G-
    element optimizer shard (31.5 GB of master/m/v traffic per step). The 1.3B model at 64
    sequences has the same flops (8*65536*1.31e9 = 6.9e14) and exactly the same optimizer
    traffic. Config 5 (70B, N=8, params + optimizer offloaded): per GPU 2.3e15 flops and
    212 GB of optimizer + 35 GB of parameter-shard host traffic per step, 1.07e-4 B/flop;
    the 1.3B model at 32 sequences with params and states on the host moves 36.7 GB per
    3.4e14 flops, the same ratio (``params_host``). The leg shows whether the offload
    hides behind compute at that ratio. Hidden fraction by the SURVEY §8(d) formula:
    1 - (t_offload - t_hbm) / t_transfer, t_transfer = host bytes / measured duplex peak;
    the traced Timeline's overlap is reported beside it."""
    import dataclasses
    import torch
    from paper_2104_07857_b200 import gpt as eg
    from paper_2104_07857_b200.comm import LocalComm
    from paper_2104_07857_b200.store import TierKind
    cfg = dataclasses.replace(eg.GPT_1P3B, batch=batch)
    peak = host_link_peak()
    bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
    steps = max(2, min(args.steps, 3))
    res = {}
    H, D = TierKind.HOST, TierKind.DEVICE
    # params on the host: the reuse cache config 5 can afford. Per GPU at config 5 (70B,
    # N=8, 4 x 1024 tokens) ~99 GB of activations and ~10 GB of rings leave ~70 GB of
    # the 180 GB for ~40 of the 87 gathered 1.61 GB layers (46 %); the same share of the
    # 1.3B model's 24 blocks is 11.
    cache = int(round(0.46 * cfg.nl)) if params_host else 0
    for name, pl in (("hbm", eg.Placement(D, D)),
                     ("offload", eg.Placement(H if params_host else D, H))):
        eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4, placement=pl,
                               param_cache=cache if name == "offload" else 0)
        for w in range(2):
            eng.step([bs[w % 2]])
        torch.cuda.synchronize()

        def host_bytes():
            return getattr(eng, "offload_bytes", 0) + getattr(eng, "fetch_bytes", 0)
        b0 = host_bytes()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for s in range(steps):
            loss = eng.step([bs[s % 2]])
        eng.flush()      # deferred optimizer-state write-back lands inside the timed region
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / steps
        res[name] = {"ms": ms, "bytes": (host_bytes() - b0) / steps, "loss": float(loss.item())}
        if name == "offload":
            eng.trace = True
            eng.step([bs[0]])
            tl = eng.timeline()
            res[name]["tl_hidden"] = tl.hidden_fraction(("pcie",))
            res[name]["pcie_busy_s"] = tl.lane_busy_s("pcie")
            sim = eng.simulated_step(duplex=True)
            res[name]["sim"] = {"measured_step_s": round(sim["measured_s"], 4),
                                "predicted_duplex_s": round(sim["predicted_s"], 4),
                                "rel_error_duplex": round(sim["rel_error"], 4)}
            eng.trace = False
        del eng
        torch.cuda.empty_cache()
    moved = res["offload"]["bytes"]
    t_xfer = moved / (peak["duplex_gbs"] * 1e9) * 1e3
    exposed = res["offload"]["ms"] - res["hbm"]["ms"]
    fl = eg.model_flops_per_step(cfg)
    what = ("config 5 per-GPU host-bytes-per-flop), bf16 params and fp32 optimizer state"
            if params_host else "config 3 per-GPU flops and optimizer traffic), fp32 optimizer state")
    return {"workload": f"GPT-1.3B x {batch} seq/GPU ({what} in pinned host DRAM",
            "ms_per_step_hbm": round(res["hbm"]["ms"], 2),
            "ms_per_step_offload": round(res["offload"]["ms"], 2),
            "tflops_offload": round(fl / (res["offload"]["ms"] / 1e3) / 1e12, 1),
            "host_bytes_per_step": int(moved),
            "param_reuse_cache_blocks": cache,
            "transfer_ms_at_duplex_peak": round(t_xfer, 2),
            "exposed_ms": round(exposed, 2),
            "hidden_fraction": round(max(0.0, 1.0 - exposed / t_xfer), 4) if t_xfer > 0 else None,
            "timeline_pcie_hidden_behind_compute": round(res["offload"]["tl_hidden"], 4),
            "timeline_pcie_busy_s": round(res["offload"]["pcie_busy_s"], 4),
            "simulator_calibration": res["offload"]["sim"],
            "loss_hbm": res["hbm"]["loss"], "loss_offload": res["offload"]["loss"]}


def _hbm_step_ms(cfg, steps: int) -> float:
    """Eager step time of ``cfg`` with every state in HBM (the offload legs' t_hbm)."""
    import torch
    from paper_2104_07857_b200 import gpt as eg
    from paper_2104_07857_b200.comm import LocalComm
    eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4)
    bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
    for w in range(2):
        eng.step([bs[w % 2]])
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in range(steps):
        eng.step([bs[s % 2]])
    t1.record()
    torch.cuda.synchronize()
    del eng
    torch.cuda.empty_cache()
    return t0.elapsed_time(t1) / steps


def config3_real_leg(args) -> dict:
    """BASELINE config 3's model itself on one GPU: GPT 10B (50 layers, hidden 4096,
    PAPER.md:677), 8 x 1024 tokens, bf16 params in HBM, all 10.3 G fp32 master / m / v
    elements (124 GB) in pinned host DRAM, streamed through the H2D || zi_rs_adam_dc ||
    D2H pipeline in the backward. At N=8 each GPU would hold 1/8 of those states; at
    N=1 the whole 247 GB of state traffic per step crosses this GPU's own host link, so
    the step is PCIe-bound by construction (the config3_equiv leg holds the N=8 per-GPU
    balance). t_hbm, for SURVEY §8(d)'s hidden fraction, cannot be measured directly
    (the states do not fit beside the activations in 180 GB): it is the linear fit
    t(nl) = a + b * nl through all-in-HBM steps of the same model at 2 and 26 layers,
    extrapolated to 50 (every block is the same work)."""
    import dataclasses
    import torch
    from paper_2104_07857_b200 import gpt as eg
    from paper_2104_07857_b200.comm import LocalComm
    from paper_2104_07857_b200.store import TierKind, _mem_available, _PinnedBuffer
    cfg = eg.GPT_10B
    P = eg.param_count(cfg)
    need = 12 * P
    avail = _mem_available() or 0
    if need > avail - _PinnedBuffer.HOST_RESERVE - (8 << 30):
        return {"skipped": f"host DRAM: {need / 2**30:.0f} GiB of pinned optimizer state "
                           f"needs more than the {avail / 2**30:.0f} GiB available"}
    peak = host_link_peak()
    steps = max(2, min(args.steps, 3))
    t_init = time.perf_counter()
    eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4,
                           placement=eg.Placement(TierKind.DEVICE, TierKind.HOST))
    init_s = time.perf_counter() - t_init
    bs = [eg.synthetic_tokens(cfg, 7, 0, s) for s in range(2)]
    eng.step([bs[0]])
    torch.cuda.synchronize()
    b0 = eng.offload_bytes
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in range(steps):
        loss = eng.step([bs[(s + 1) % 2]])
    eng.flush()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    moved = (eng.offload_bytes - b0) / steps
    eng.trace = True
    eng.step([bs[0]])
    tl = eng.timeline()
    eng.trace = False
    loss = float(loss.item())
    eng.close()
    del eng
    torch.cuda.empty_cache()
    t2 = _hbm_step_ms(dataclasses.replace(cfg, nl=2), steps)
    t26 = _hbm_step_ms(dataclasses.replace(cfg, nl=26), steps)
    t_hbm = t2 + (t26 - t2) * (cfg.nl - 2) / 24
    t_xfer = moved / (peak["duplex_gbs"] * 1e9) * 1e3
    exposed = ms - t_hbm
    fl = eg.model_flops_per_step(cfg)
    return {"workload": "GPT-10B (50 x 4096, BASELINE config 3's model) at N=1, 8 x 1024 tokens, "
                        "bf16 params in HBM, fp32 master / m / v (all 10.3 G elements) in pinned "
                        "host DRAM",
            "params": P, "pinned_state_bytes": need, "engine_init_s": round(init_s, 1),
            "ms_per_step_offload": round(ms, 1),
            "tflops_offload": round(fl / (ms / 1e3) / 1e12, 1),
            "loss": loss,
            "host_bytes_per_step": int(moved),
            "host_link_gbs": round(moved / (ms / 1e3) / 1e9, 1),
            "host_link_peak": peak,
            "ms_per_step_hbm_fit": round(t_hbm, 1),
            "hbm_fit_points_ms": {"nl2": round(t2, 2), "nl26": round(t26, 2)},
            "tflops_hbm_fit": round(fl / (t_hbm / 1e3) / 1e12, 1),
            "transfer_ms_at_duplex_peak": round(t_xfer, 1),
            "exposed_ms": round(exposed, 1),
            "hidden_fraction": round(max(0.0, 1.0 - exposed / t_xfer), 4),
            "timeline_pcie_hidden_behind_compute": round(tl.hidden_fraction(("pcie",)), 4),
            "timeline_pcie_busy_s": round(tl.lane_busy_s("pcie"), 3),
            "bound": "host link (N=1 carries all 8 ranks' state traffic)"}


def _leg_subprocess(name: str, args, timeout: int = 1200) -> dict:
    """Run one heavy leg in a fresh process (its pinned memory is the host's, and a
    failure cannot take the main line with it); the child prints one JSON object."""
    import gc
    import subprocess
    import torch
    gc.collect()                 # engines of earlier legs hold pinned arenas through cycles
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch._C._host_emptyCache()  # and torch's pinned host cache (host_link_peak buffers)
    cmd = [sys.executable, os.path.abspath(__file__), "--leg", name,
           "--steps", str(args.steps), "--warmup", str(args.warmup)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"error": f"leg {name} timed out after {timeout} s"}
    for line in reversed(r.stdout.strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return {"error": f"leg {name} exited {r.returncode}: {r.stderr.strip()[-300:]}"}


def disk_peak(root: str, nbytes: int = 2 << 30) -> dict:
    """O_DIRECT write then read of one file through the native engine (8 threads,
    8 MiB pieces): the disk's own sequential bandwidth, the NVMe legs' denominator."""
    import os as _os
    from paper_2104_07857_b200.aio import AioEngine
    from paper_2104_07857_b200.store import _PinnedBuffer
    buf = _PinnedBuffer(256 << 20)
    path = _os.path.join(root, "zinf_disk_peak.bin")
    eng = AioEngine(8)
    try:
        fds = eng.open(path, write=True, create=True)
        res = {}
        for name, write in (("write_gbs", True), ("read_gbs", False)):
            t = time.perf_counter()
            ids = [eng.submit(fds, write, buf.ptr, o, o + (256 << 20))
                   for o in range(0, nbytes, 256 << 20)]
            for i in ids:
                eng.wait(i)
            res[name] = round(nbytes / (time.perf_counter() - t) / 1e9, 2)
        AioEngine.close_file(fds)
    finally:
        eng.close()
        buf.free()
        if _os.path.exists(path):
            _os.unlink(path)
    return res


def nvme_params_leg(cfg, args, bs, steps) -> dict:
    """ZeRO-Infinity's defining placement (PAPER §6.2): the 1.3B step with the bf16
    parameter shards as reference-format .shard files in the NVMe tier and the fp32
    optimizer states in pinned host DRAM. Every fetch position runs the plan's three
    stages: nc (NVMe -> pinned, store workers) issued 3 positions
    ahead, cg (pinned -> HBM, H2D stream) 2 ahead, gg (gather) 1 ahead; updated bf16
    params are written back to their files. Hidden fraction by SURVEY §8(d):
    1 - (t_nvme - t_hbm) / t_transfer, t_transfer = the step's host-link bytes at the
    measured duplex peak (the nc reads come from files the page cache holds on this
    box, so PCIe, not the disk, carries the transfer)."""
    import shutil
    import tempfile
    import torch
    from paper_2104_07857_b200 import gpt as eg
    from paper_2104_07857_b200.comm import LocalComm
    from paper_2104_07857_b200.store import TierKind
    peak = host_link_peak()
    res = {}
    root = tempfile.mkdtemp(prefix="zinf_nvme_params_", dir=args.nvme_dir)
    try:
        for name, pl in (("hbm", eg.Placement(TierKind.DEVICE, TierKind.DEVICE)),
                         ("nvme", eg.Placement(TierKind.NVME, TierKind.HOST))):
            eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4, placement=pl,
                                   nvme_root=root if name == "nvme" else None)
            for w in range(2):
                eng.step([bs[w % 2]])
            eng.flush()
            torch.cuda.synchronize()

            def counters():
                return (getattr(eng, "offload_bytes", 0) + getattr(eng, "fetch_bytes", 0),
                        getattr(eng, "nc_bytes", 0))
            h0, n0 = counters()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t = time.perf_counter()
            t0.record()
            for s in range(steps):
                loss = eng.step([bs[s % 2]])
            eng.flush()
            t1.record()
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t) * 1e3 / steps
            h1, n1 = counters()
            res[name] = {"ms": t0.elapsed_time(t1) / steps, "wall_ms": wall,
                         "host_bytes": (h1 - h0) / steps, "nc_bytes": (n1 - n0) / steps,
                         "loss": float(loss.item())}
            if name == "nvme":
                eng.trace = True
                eng.step([bs[0]])
                eng.flush()
                tl = eng.timeline()
                res[name]["tl_hidden"] = tl.hidden_fraction(("pcie",))
                eng.trace = False
            eng.close()
            del eng
            torch.cuda.empty_cache()
    finally:
        shutil.rmtree(root, ignore_errors=True)
    nv, hb = res["nvme"], res["hbm"]
    t_xfer = nv["host_bytes"] / (peak["duplex_gbs"] * 1e9) * 1e3
    exposed = nv["ms"] - hb["ms"]
    return {"workload": "GPT-1.3B ZeRO-Infinity step: bf16 params as NVMe-tier .shard files "
                        "(nc -> cg -> gg at plan depths 3 / 2 / 1), fp32 optimizer state in "
                        "pinned host DRAM",
            "ms_per_step_hbm": round(hb["ms"], 2), "ms_per_step_nvme": round(nv["ms"], 2),
            "wall_ms_per_step_nvme": round(nv["wall_ms"], 2),
            "tflops_nvme": round(eg.model_flops_per_step(cfg) / (nv["ms"] / 1e3) / 1e12, 1),
            "nc_bytes_per_step": int(nv["nc_bytes"]),
            "host_bytes_per_step": int(nv["host_bytes"]),
            "transfer_ms_at_duplex_peak": round(t_xfer, 2),
            "exposed_ms": round(exposed, 2),
            "hidden_fraction": round(max(0.0, 1.0 - exposed / t_xfer), 4) if t_xfer > 0 else None,
            "timeline_pcie_hidden_behind_compute": round(nv["tl_hidden"], 4),
            "loss_hbm": hb["loss"], "loss_nvme": nv["loss"],
            "losses_bitwise_equal": hb["loss"] == nv["loss"]}


def nvme_leg(cfg, args, bs, steps, direct: bool = False) -> dict:
    """The 1.3B step with fp32 master/m/v as .shard files in the NVMe tier (PAPER §6.2):
    per bucket the streamer runs nc-read -> H2D -> zi_rs_adam_dc -> D2H -> nc-write in
    chunks. Files go through the OS page cache (the shard header is 20 B, so payloads
    are not O_DIRECT-aligned); the box's disk is a virtio block device."""
    import shutil
    import tempfile
    import torch
    from paper_2104_07857_b200 import gpt as eg
    from paper_2104_07857_b200.comm import LocalComm
    from paper_2104_07857_b200.store import TierKind
    root = tempfile.mkdtemp(prefix="zinf_nvme_", dir=args.nvme_dir)
    try:
        eng = eg.GPTZeroEngine(cfg, LocalComm(1), seed=7, lr=1e-4, nvme_root=root,
                               placement=eg.Placement(TierKind.DEVICE, TierKind.NVME),
                               nvme_direct=direct)
        eng.step([bs[0]])
        torch.cuda.synchronize()
        b0 = eng.streamer.bytes
        t = time.perf_counter()
        for s in range(steps):
            loss = eng.step([bs[s % 2]])
        loss.item()
        ms = (time.perf_counter() - t) * 1e3 / steps
        moved = (eng.streamer.bytes - b0) / steps
        how = ("native engine: O_DIRECT whole blocks, C worker threads" if direct else
               "Python store workers through the OS page cache")
        out = {"workload": "GPT-1.3B ZeRO-3 step, fp32 optimizer state (15.8 GB) in NVMe-tier "
                           f".shard files ({how})",
               "nvme_root": args.nvme_dir or tempfile.gettempdir(),
               "ms_per_step": round(ms, 1),
               "tflops": round(eg.model_flops_per_step(cfg) / (ms / 1e3) / 1e12, 2),
               "nvme_bytes_per_step": int(moved),
               "nvme_gbs": round(moved / (ms / 1e3) / 1e9, 2),
               "timing": "host wall clock around step() (the step ends with a host drain)"}
        if direct:
            peak = disk_peak(root)
            out["disk_peak"] = peak
            both = 1.0 / (0.5 / peak["read_gbs"] + 0.5 / peak["write_gbs"])
            out["frac_of_disk_serial_rw"] = round(out["nvme_gbs"] / both, 3)
        eng.close()
        del eng
    finally:
        shutil.rmtree(root, ignore_errors=True)
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-offload", action="store_true", help="skip the optimizer-offload leg")
    ap.add_argument("--no-graph", action="store_true", help="eager steps instead of the CUDA graph")
    ap.add_argument("--no-nvme", action="store_true", help="skip the NVMe optimizer-state leg")
    ap.add_argument("--nvme-dir", default=None, help="directory for the NVMe leg's shard files")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-config3", action="store_true", help="skip the real 10B offload leg")
    ap.add_argument("--leg", default=None, choices=["config3_real"],
                    help="run one heavy leg alone and print its JSON object")
    args = ap.parse_args()
    sys.path.insert(0, ROOT)
    if args.leg == "config3_real":
        import torch
        torch.cuda.set_device(0)
        print(json.dumps(_safe(config3_real_leg, args)), flush=True)
        return 0
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}",
              file=sys.stderr)
        return 2
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


def spawn_ranks(args) -> int:
    """--gpus N without a launcher: start N ranks through torch.distributed.run (one
    process per GPU, rendezvous on 127.0.0.1). With fewer GPUs than N on the box the
    ranks time-share cuda:0 (ZINF_BENCH_SAME_GPU=1; the line says same_gpu / physical_gpus)."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    try:
        import torch
        ndev = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        ndev = 0
    if ndev < args.gpus:
        env["ZINF_BENCH_SAME_GPU"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    sys.exit(main())
