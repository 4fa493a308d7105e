"""The real multi-process path (DistComm) on one GPU: 2 processes, CUDA-IPC-mapped peer buffers.

Each process is one rank with its own CUDA context on cuda:0; torch.distributed
(gloo) carries only the IPC handles, and the data path is exactly the
multi-GPU one: P2P gather of peers' bf16 shards, zi_barrier over IPC flag
words, zi_rs_adam folding the peers' gradient buckets in rank order. The
result must equal the single-process LocalComm(2) run of the same data bit for bit
(the step is deterministic: fixed-order attention / embedding backward, rank-order RS).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _placement(name):
    from paper_2104_07857_b200.gpt import Placement
    from paper_2104_07857_b200.store import TierKind
    D, H, V = TierKind.DEVICE, TierKind.HOST, TierKind.NVME
    return {"hbm": Placement(D, D), "params_host": Placement(H, D), "all_host": Placement(H, H),
            "params_nvme": Placement(V, H)}[name]


def _rank_main(rank, world, port, q, placement="hbm", graph=False, cache=0):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2104_07857_b200 import gpt as eg
        from paper_2104_07857_b200.comm import DistComm
        c = eg.GPTConfig(nl=2, hd=128, heads=2, seq=128, vocab=256, batch=2)
        comm = DistComm()
        eng = eg.GPTZeroEngine(c, comm, lr=1e-3, placement=_placement(placement),
                               offload_chunk=20_000, param_cache=cache)
        losses = []
        run = eng.step_graphed if graph else eng.step
        for step in range(2):
            losses.append(run([eg.synthetic_tokens(c, 7, rank, step)]).item())
        torch.cuda.synchronize()
        out = {k: eng.shard(k, 0)["p32"].cpu().numpy() for k in eng.by_key}
        if eng.nvme_params:   # the bf16 param files hold the update (nc lane, both ways)
            for k in eng.by_key:
                assert torch.equal(eng.param_file_shard(k, 0).view(torch.int16),
                                   eng.shard(k, 0)["p16"].view(torch.int16)), k
            eng.close()
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, losses, out))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("placement,graph,cache", [("hbm", False, 0), ("params_host", False, 0),
                                                   ("all_host", False, 0), ("hbm", True, 0),
                                                   ("params_host", True, 0),
                                                   ("params_host", False, 1),
                                                   ("params_nvme", False, 0)])
def test_two_processes_match_local_comm(placement, graph, cache):
    """graph=True: each rank captures its step (P2P gathers, barriers with device-side
    epochs, RS + Adam over peer buckets) in a CUDA graph and replays it."""
    from paper_2104_07857_b200 import gpt as eg
    from paper_2104_07857_b200.comm import LocalComm
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, placement, graph, cache))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, a, b = q.get(timeout=600)
        assert a != "error", b
        res[r] = (a, b)
    for p in procs:
        p.join(timeout=60)
    c = eg.GPTConfig(nl=2, hd=128, heads=2, seq=128, vocab=256, batch=2)
    ref = eg.GPTZeroEngine(c, LocalComm(world), lr=1e-3)
    ref_losses = [ref.step([eg.synthetic_tokens(c, 7, r, step) for r in range(world)]).item()
                  for step in range(2)]
    for r in range(world):
        dist_losses, shards = res[r]
        # DistComm returns each rank's own loss; LocalComm the mean
        for key, arr in shards.items():
            want = ref.shard(key, r)["p32"].cpu().numpy()
            assert arr.shape == want.shape
            assert np.array_equal(arr.view(np.uint32), want.view(np.uint32)), key   # bitwise
    mean_dist = [(res[0][0][s] + res[1][0][s]) / 2 for s in range(2)]
    np.testing.assert_allclose(mean_dist, ref_losses, rtol=1e-6)


def _oracle_rank_main(rank, world, port, q, gemm_select):
    """BASELINE config 1 with one process per rank: per-step loss, gradient shards and
    master shards (before / after) for the oracle comparison in the parent."""
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2104_07857_b200 import gpt as eg
        from paper_2104_07857_b200.comm import DistComm
        comm = DistComm()
        eng = eg.GPTZeroEngine(eg.TINY, comm, lr=1e-3, gemm_select=gemm_select)
        eng.capture_grads = True
        out = []
        for step in range(3):
            loss = eng.step([eg.synthetic_tokens(eg.TINY, 7, rank, step)]).item()
            out.append((loss, {k: v[rank].cpu().numpy() for k, v in eng.grad_shards.items()},
                        {k: eng.shard(k, 0)["p32"].cpu().numpy() for k in eng.by_key}))
        torch.cuda.synchronize()
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, "ok", out))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("gemm_select", ["cublas", "zi"])
def test_config1_two_processes_match_oracle(gemm_select):
    """BASELINE config 1 (nl4 / hd256 / seq128 / batch4 / V512) at world 2 with one
    process per rank (DistComm: P2P gathers, stream-memop barriers, RS + Adam over the
    peer's gradient bucket), 3 steps against the CPU oracle with test_gpt_gpu's
    tolerances; gemm_select="zi" runs every linear on the tcgen05 GEMM (no SM is held
    by a waiting barrier, so a time-sliced peer cannot be starved)."""
    from oracle import gpt as og
    from oracle import numerics as nx
    from paper_2104_07857_b200 import gpt as eg
    from test_gpt_gpu import TOL_BF16, rel
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_oracle_rank_main, args=(r, world, port, q, gemm_select))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, st, b = q.get(timeout=600)
        assert st == "ok", b
        res[r] = b
    for p in procs:
        p.join(timeout=60)
    c = eg.TINY
    ost = og.init_partitioned(og.GPTConfig(c.nl, c.hd, c.heads, c.seq, c.vocab, c.batch), world,
                              half_kind=nx.HALF_BF16)
    lr = 1e-3
    for step in range(3):
        prev = {k: [s.astype(np.float64) for s in ost.p32[k]] for k in ost.p32}
        bs = [tuple(t.cpu().numpy() for t in eg.synthetic_tokens(c, 7, r, step, device="cpu"))
              for r in range(world)]
        oloss, gsh = og.train_step(ost, bs, lr=lr)
        mean = (res[0][step][0] + res[1][step][0]) / 2   # DistComm: each rank's own loss
        assert abs(mean - oloss) <= TOL_BF16[0] * abs(oloss), (step, mean, oloss)
        errs, num, den = [], 0.0, 0.0
        for r in range(world):
            _, g, p32 = res[r][step]
            for key in gsh:
                assert rel(g[key], gsh[key][r]) < TOL_BF16[1], (step, key, r)
                dg = p32[key].astype(np.float64) - prev[key][r]
                do = ost.p32[key][r].astype(np.float64) - prev[key][r]
                errs.append(np.abs(dg - do) / lr)
                num += float(((dg - do) ** 2).sum())
                den += float((do ** 2).sum())
        e = np.concatenate(errs)
        assert (e > 0.1).mean() < TOL_BF16[2] and np.sqrt(num / den) < TOL_BF16[3], step


def _ctx_rank_main(rank, world, port, q):
    """zi_ctx collectives through DistComm windows: one rank per process."""
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import numerics as nx
        from paper_2104_07857_b200.comm import DistComm
        comm = DistComm()
        n = 10_007                                   # ragged: last shard zero padded
        L = -(-n // world)
        off = 24                                     # window at an offset inside its allocation
        rng = np.random.default_rng(100 + rank)
        g_bits = nx.f32_to_half_bits(rng.standard_normal(n).astype(np.float32), nx.HALF_BF16)
        buf = comm.alloc((off + n,), torch.bfloat16)
        grads = buf[off:]
        grads.copy_(torch.from_numpy(g_bits.view(np.int16).copy()).view(torch.bfloat16))
        pbuf = comm.alloc((L,), torch.float32)
        pbuf.copy_(torch.arange(rank * L, rank * L + L, dtype=torch.float32) * 0.5)
        comm.share(grads)
        comm.share(pbuf)
        comm.device_barrier()                        # peers' windows are written
        out = torch.empty(L, dtype=torch.float32, device="cuda")
        comm.reduce_scatter_window(grads, L, out, scale=1.0 / world)
        full = torch.empty(n, dtype=torch.float32, device="cuda")
        comm.allgather_window(pbuf, L, full)
        full_ce = torch.empty(n, dtype=torch.float32, device="cuda")
        comm.allgather_window(pbuf, L, full_ce, use_copy_engine=True)
        comm.device_barrier()                        # peers are done reading our windows
        torch.cuda.synchronize()
        info = [ctypes_info(comm)]
        res = (out.cpu().numpy(), full.cpu().numpy(), full_ce.cpu().numpy(), g_bits, info)
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, "ok", res))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, "error", traceback.format_exc()))


def ctypes_info(comm):
    import ctypes
    from paper_2104_07857_b200 import _lib
    r, w, d = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.call("zi_ctx_info", comm.ctx, ctypes.byref(r), ctypes.byref(w), ctypes.byref(d))
    return r.value, w.value, d.value


def test_ctx_collectives_two_processes():
    """zi_ctx_reduce_scatter_cast / zi_ctx_allgather across 2 processes:
    RS bit-exact against the oracle's rank-order fold, gathers bit-exact (SM kernel and
    copy engines), windows at byte offsets inside their allocations."""
    from oracle import numerics as nx
    from oracle.partition import reduce_scatter_cast
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_ctx_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, st, b = q.get(timeout=300)
        assert st == "ok", b
        res[r] = b
    for p in procs:
        p.join(timeout=60)
    n, L = 10_007, 5004
    contribs = [nx.half_bits_to_f32(res[r][3], nx.HALF_BF16) for r in range(world)]
    want = reduce_scatter_cast(contribs, world, 1.0 / world)
    pfull = (np.arange(world * L, dtype=np.float32) * 0.5)[:n]
    for r in range(world):
        out, full, full_ce, _, info = res[r]
        assert info[0] == (r, world, 0)
        assert np.array_equal(out.view(np.uint32), want[r].view(np.uint32))
        assert np.array_equal(full, pfull) and np.array_equal(full_ce, pfull)
