"""The SPEC collectives with one process per rank (DistComm), 2 processes on one GPU.

Each rank holds only its own shards (its own TierStore), as with one process
per GPU; the peers' shards are read over CUDA-IPC-mapped windows (NVLink on a
multi-GPU box). Everything is compared with the CPU oracle (oracle/partition.py,
oracle/tiling.py, the simulated-rank run of the same SPEC harness):

* partition -> allgather over the DEVICE / HOST / NVME tiers, four dtypes,
  ragged lengths, SM-kernel and copy-engine gathers: bit-exact;
* reduce_scatter with one and with two gradient groups per rank (bf16 -> fp32,
  f32, f64): bit-exact against the rank-major sequential fold;
* broadcast_fetch from an owner rank == allgather result, bytes on one path;
* forward_tiled / backward_tiled with just-in-time tile gathers across the two
  processes == the single-process run, bit for bit;
* run_training (AC-9): the 2-process digest and losses == the simulated world-1
  and world-2 runs, bit for bit.

Both barrier flavours run: stream write/wait-value (the default, no SM held) and
the spin kernel with a device-side epoch.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

DTYPES = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32, "f64": torch.float64}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _values(n, dtype, seed):
    x = np.random.default_rng(seed).standard_normal(n).astype(np.float32)
    return torch.from_numpy(x).to(dtype)


def _bits(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu().contiguous()
    w = t.element_size()
    return t.view({2: torch.int16, 4: torch.int32, 8: torch.int64}[w]).numpy()


def _harness_spec():
    from paper_2104_07857_b200 import harness as H
    L = H.LayerSpec
    return H.ModelSpec([L("linear", 8, 16, "relu"), L("tiled_linear", 16, 16, "gelu-approx", tiles=4),
                        L("linear", 16, 16, "relu"), L("linear", 16, 16, "relu"),
                        L("linear", 16, 4)], tied_pairs=[(2, 3)], seed=7)


def _rank_main(rank, world, port, q, tmp, barrier_kind):
    import faulthandler
    import time
    log = open(os.path.join(tmp, f"progress_r{rank}.log"), "w", buffering=1)
    faulthandler.dump_traceback_later(240, exit=True, file=log)

    def say(*a):
        print(f"{time.time():.3f}", *a, file=log, flush=True)
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ZI_BARRIER=barrier_kind)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2104_07857_b200 import harness as H
        from paper_2104_07857_b200 import tiling as T
        from paper_2104_07857_b200.comm import DistComm
        from paper_2104_07857_b200.partition import (allgather, broadcast_fetch, partition,
                                                      reduce_scatter)
        from paper_2104_07857_b200.store import TierKind, TierStore
        comm = DistComm()
        assert comm.barrier_kind == barrier_kind
        res = {}
        store = TierStore(1 << 30, 1 << 30, nvme_root=os.path.join(tmp, f"r{rank}"))
        # -- partition -> allgather
        for tier in (TierKind.DEVICE, TierKind.HOST, TierKind.NVME):
            for name, dt in DTYPES.items():
                for n in (1, 7, 10_007):
                    full = _values(n, dt, n)
                    pt = partition(full.cuda(), world, tier, store, key=f"ag.{tier.value}.{name}.{n}",
                                   comm=comm)
                    mine = store.keys(tier)
                    assert f"{pt.key}/rank{rank}" in mine and f"{pt.key}/rank{1 - rank}" not in mine
                    sm = allgather(pt, store, comm)
                    ce = allgather(pt, store, comm, use_copy_engine=True)
                    res[("ag", tier.value, name, n)] = (_bits(sm), _bits(ce))
            say("allgather", tier.value)
        # -- reduce_scatter: k gradient groups per rank, folded rank-major
        for name, dt in (("bf16", torch.bfloat16), ("f32", torch.float32), ("f64", torch.float64)):
            for k in (1, 2):
                n = 4099
                mine = [_values(n, dt, 1000 + rank * k + j).cuda() for j in range(k)]
                out = reduce_scatter(mine, world, comm=comm, scale=0.25)
                assert len(out) == 1
                res[("rs", name, k)] = _bits(out[0])
                say("reduce_scatter", name, k)
        # -- broadcast_fetch from owner rank 1 vs allgather
        full = _values(5000, torch.bfloat16, 77)
        if rank == 1:
            store.write("bc.w", full.cuda(), TierKind.HOST).wait()
        got, charged = broadcast_fetch("bc.w", TierKind.HOST, store, comm=comm, owner=1,
                                       numel=5000, dtype=torch.bfloat16)
        res["bc"] = (_bits(got), charged)
        say("broadcast_fetch")
        # -- tiled linear with just-in-time gathers across processes (bf16 tcgen05 tiles)
        g = torch.Generator().manual_seed(3)
        M, K, Nout = 256, 512, 1024
        W = (torch.randn(Nout, K, generator=g) * K ** -0.5).bfloat16().cuda()
        b = torch.randn(Nout, generator=g).bfloat16().cuda()
        x = torch.randn(M, K, generator=g).bfloat16().cuda()
        gy = torch.randn(M, Nout, generator=g).bfloat16().cuda()
        tl = T.tile_linear(W, b, 4, store, TierKind.DEVICE, key="tl", world_size=world, comm=comm)
        for prefetch in (False, True):
            y = T.forward_tiled(tl, x, store, comm=comm, prefetch=prefetch)
            dW, db, dx = T.backward_tiled(tl, x, gy, store, comm=comm, prefetch=prefetch)
            res[("tile", prefetch)] = (_bits(y), [_bits(d) for d in dW], [_bits(d) for d in db],
                                      _bits(dx))
            say("tiling", prefetch)
        # -- the SPEC harness, data parallel over the two processes (AC-9)
        s = _harness_spec()
        for pl in ("device", "nvme"):
            kind = TierKind.DEVICE if pl == "device" else TierKind.NVME
            with TierStore(1 << 30, 1 << 30, nvme_root=os.path.join(tmp, f"h{pl}{rank}")) as st:
                res[("ac9", pl)] = H.run_training(s, world, H.HarnessPlacement.all(kind), 8, 7, st,
                                                  chunk_elems=5, comm=comm)
            say("ac9", pl)
        torch.cuda.synchronize()
        dist.barrier()
        store.close()
        comm.close()
        dist.destroy_process_group()
        say("done")
        faulthandler.cancel_dump_traceback_later()
        q.put((rank, "ok", res))
    except Exception:  # noqa: BLE001
        import traceback
        say(traceback.format_exc())
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("barrier_kind", ["memop", "kernel"])
def test_spec_collectives_two_processes(tmp_path, barrier_kind):
    from oracle import numerics as nx
    from oracle import partition as op
    from paper_2104_07857_b200 import harness as H
    from paper_2104_07857_b200 import tiling as T
    from paper_2104_07857_b200.comm import LocalComm
    from paper_2104_07857_b200.store import TierKind, TierStore
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, str(tmp_path), barrier_kind))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    import queue
    for _ in range(world):
        try:
            r, st, b = q.get(timeout=300)
        except queue.Empty:
            logs = [open(tmp_path / f"progress_r{r}.log").read() for r in range(world)]
            for p in procs:
                p.kill()
            pytest.fail("rank timed out:\n" + "\n".join(logs))
        assert st == "ok", b
        res[r] = b
    for p in procs:
        p.join(timeout=60)
    # allgather: bit-exact oracle round trip on every rank, every tier / dtype / length
    for name, dt in DTYPES.items():
        for n in (1, 7, 10_007):
            full = _values(n, dt, n)
            want = _bits(torch.from_numpy(np.ascontiguousarray(
                op.allgather(op.partition(_bits(full), world), n))).view(dt))
            for tier in ("device", "host", "nvme"):
                for r in range(world):
                    sm, ce = res[r][("ag", tier, name, n)]
                    assert np.array_equal(sm, want) and np.array_equal(ce, want), (tier, name, n, r)
    # reduce_scatter: rank-major sequential fold (rank 0's groups, then rank 1's)
    for name, dt in (("bf16", torch.bfloat16), ("f32", torch.float32), ("f64", torch.float64)):
        acc = np.float64 if dt == torch.float64 else np.float32
        for k in (1, 2):
            n, L = 4099, 2050
            s = np.zeros(L * world, acc)
            for g in range(world * k):
                c = _values(n, dt, 1000 + g)
                s[:n] = s[:n] + c.to(torch.float64 if dt == torch.float64 else torch.float32).numpy()
            for r in range(world):
                want = (s[r * L:(r + 1) * L] * acc(0.25)).astype(acc)
                assert np.array_equal(res[r][("rs", name, k)], want.view(
                    np.int64 if acc == np.float64 else np.int32)), (name, k, r)
    # broadcast_fetch: the owner's whole tensor on every rank, charged to one path
    full = _bits(_values(5000, torch.bfloat16, 77))
    for r in range(world):
        got, charged = res[r]["bc"]
        assert np.array_equal(got, full) and charged == 5000 * 2 * (world - 1)
    # tiling: the 2-process run == the single-process simulated world-2 run, bit for bit
    g = torch.Generator().manual_seed(3)
    M, K, Nout = 256, 512, 1024
    W = (torch.randn(Nout, K, generator=g) * K ** -0.5).bfloat16().cuda()
    b = torch.randn(Nout, generator=g).bfloat16().cuda()
    x = torch.randn(M, K, generator=g).bfloat16().cuda()
    gy = torch.randn(M, Nout, generator=g).bfloat16().cuda()
    with TierStore(1 << 30, 1 << 30, nvme_root=str(tmp_path / "local")) as st:
        tl = T.tile_linear(W, b, 4, st, TierKind.DEVICE, key="tl", world_size=world)
        y = _bits(T.forward_tiled(tl, x, st))
        dW, db, dx = T.backward_tiled(tl, x, gy, st)
        for r in range(world):
            for prefetch in (False, True):
                ry, rdW, rdb, rdx = res[r][("tile", prefetch)]
                assert np.array_equal(ry, y)
                assert all(np.array_equal(a, _bits(d)) for a, d in zip(rdW, dW))
                assert all(np.array_equal(a, _bits(d)) for a, d in zip(rdb, db))
                assert np.array_equal(rdx, _bits(dx))
    # AC-9 across processes: digest and losses equal the simulated runs
    s = _harness_spec()
    with TierStore(1 << 30, 1 << 30, nvme_root=str(tmp_path / "h1")) as st:
        d1, l1 = H.run_training(s, 1, H.HarnessPlacement.all(TierKind.DEVICE), 8, 7, st)
    with TierStore(1 << 30, 1 << 30, nvme_root=str(tmp_path / "h2")) as st:
        d2, l2 = H.run_training(s, 2, H.HarnessPlacement.all(TierKind.DEVICE), 8, 7, st,
                                comm=LocalComm(2))
    assert d1 == d2 and l1 == l2
    for r in range(world):
        for pl in ("device", "nvme"):
            dr, lr = res[r][("ac9", pl)]
            assert dr == d1, (r, pl)
            assert lr == l1, (r, pl)
