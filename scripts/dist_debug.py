"""2-process DistComm smoke with progress logs (one GPU): python scripts/dist_debug.py memop|kernel.

Each rank writes gpurun_out/dist_debug_<kind>_r<rank>.log as it passes each stage, and
faulthandler dumps every thread's stack if a stage hangs.
"""

import faulthandler
import os
import socket
import sys
import time

import torch
import torch.multiprocessing as mp

sys.path.insert(0, ".")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def rank_main(rank, world, port, kind):
    log = open(f"gpurun_out/dist_debug_{kind}_r{rank}.log", "w", buffering=1)
    faulthandler.dump_traceback_later(40, exit=True, file=log)

    def say(*a):
        print(f"{time.time():.3f}", *a, file=log, flush=True)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ZI_BARRIER=kind)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2104_07857_b200.comm import DistComm
    from paper_2104_07857_b200.partition import allgather, partition
    from paper_2104_07857_b200.store import TierKind, TierStore
    comm = DistComm()
    say("comm", comm.barrier_kind)
    comm.open_channels((0,))
    say("channel open")
    for i in range(4):
        comm.device_barrier()
        torch.cuda.synchronize()
        say("barrier", i)
    store = TierStore(1 << 30, 1 << 30, nvme_root=f"/tmp/dd{rank}")
    full = torch.arange(1001, dtype=torch.float32, device="cuda")
    pt = partition(full, world, TierKind.DEVICE, store, key="x", comm=comm)
    say("partitioned")
    out = allgather(pt, store, comm)
    torch.cuda.synchronize()
    say("gathered", bool(torch.equal(out, full)))
    import numpy as np
    for tier in (TierKind.DEVICE, TierKind.HOST):
        for dt in (torch.bfloat16, torch.float32):
            for n in (1, 7, 10007):
                full = torch.from_numpy(np.random.default_rng(n).standard_normal(n).astype(np.float32)).to(dt)
                pt = partition(full.cuda(), world, tier, store, key=f"ag.{tier.value}.{dt}.{n}", comm=comm)
                torch.cuda.synchronize()
                say("part", tier.value, dt, n)
                stage, _ = comm.staging(f"ag:{pt.key}", pt.shard_len, pt.dtype)
                torch.cuda.synchronize()
                say("staged")
                comm.device_barrier(channel=3)
                torch.cuda.synchronize()
                say("barrier ch3", comm._bar_count)
                sm = allgather(pt, store, comm)
                torch.cuda.synchronize()
                say("ag sm", bool(torch.equal(sm.cpu(), full)))
                ce = allgather(pt, store, comm, use_copy_engine=True)
                torch.cuda.synchronize()
                say("ag ce", bool(torch.equal(ce.cpu(), full)))
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    say("done")
    faulthandler.cancel_dump_traceback_later()


if __name__ == "__main__":
    kind = sys.argv[1]
    os.makedirs("gpurun_out", exist_ok=True)
    port = _port()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=rank_main, args=(r, 2, port, kind)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=90)
        if p.is_alive():
            p.kill()
    print(kind, [p.exitcode for p in ps])
