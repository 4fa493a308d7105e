"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host plumbing.

Each rank materialises only its own shard (``partition`` with a DistComm
writes ``key/rank<r>`` for its own rank), the per-rank shards reassemble
bit-exactly into the oracle's gather, the rank-order reduce-scatter layout
matches the oracle, and DistComm's object / max collectives work.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nvme_root, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.partition import allgather as o_ag, partition as o_part, reduce_scatter as o_rs
        from paper_2104_07857_b200.comm import DistComm
        from paper_2104_07857_b200.partition import make_shard, partition, shard_len
        from paper_2104_07857_b200.store import TierKind, TierStore
        comm = DistComm()
        assert (comm.rank, comm.world) == (rank, world)
        assert comm.all_gather_object(rank * 10) == [r * 10 for r in range(world)]
        assert comm.allreduce_max(float(rank)) == float(world - 1)
        n = 1001
        full = torch.from_numpy(np.random.default_rng(5).standard_normal(n).astype(np.float32))
        st = TierStore(0, 1 << 20, nvme_root=os.path.join(nvme_root, f"r{rank}"), sync_io=True)
        pt = partition(full, world, TierKind.HOST, st, key="w", comm=comm)
        assert st.keys(TierKind.HOST) == [f"w/rank{rank}"]            # own shard only
        mine = st.tensor(f"w/rank{rank}", TierKind.HOST)
        assert np.array_equal(mine.numpy(), o_part(full.numpy(), world)[rank])
        parts = [torch.empty(pt.shard_len) for _ in range(world)]
        dist.all_gather(parts, mine.contiguous())
        assert np.array_equal(o_ag([p.numpy() for p in parts], n), full.numpy())
        # reduce-scatter layout: rank r owns [r*L, (r+1)*L) of the rank-order sum
        contrib = torch.from_numpy(np.random.default_rng(100 + rank).standard_normal(n).astype(np.float32))
        allc = [torch.empty(n) for _ in range(world)]
        dist.all_gather(allc, contrib)
        want = o_rs([c.numpy() for c in allc], world)[rank]
        L = shard_len(n, world)
        s = torch.zeros(L)
        for c in allc:                                       # fold in rank order
            s = s + make_shard(c, world, rank)
        assert np.array_equal(s.numpy(), want)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_two_rank_partition_and_collectives(tmp_path):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
