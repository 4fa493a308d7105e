"""NVMe-resident optimizer states for the GPT engine (PAPER §5.1.1, §6.2 "nc-transfer").

The fp32 master / m / v shards of every bucket live in the TierStore's NVMe
tier (one ``.shard`` file per key, the reference format, store.py:10-18).
When a bucket's gradients are complete, a dedicated streamer thread runs the
chunk pipeline (depth ``slots``):

    nc   store.read_into(file range -> pinned R[k])      store worker threads
    cg   pinned R[k] -> HBM staging S[k]                  h2d stream
         zi_rs_adam_dc(contributions, S[k]) -> p16        optimizer stream
         HBM S[k] -> pinned W[k]                          d2h stream
    nc   store.write_from(pinned W[k] -> file range)      store worker threads

Reads of chunks c+1 .. c+slots-1 are in flight while chunk c computes; a
pinned slot is refilled only after its previous H2D / file write finished.
The thread keeps the compute stream free of host waits: the engine's main
thread only waits for a bucket's "gradient slot free" event before it
overwrites that slot, and for the whole queue at the end of the step.
"""

from __future__ import annotations

import queue
import threading

import torch

from . import kernels
from .store import TierKind, TierStore

STATES = ("p32", "m", "v")


class NvmeOptimizerStreamer:
    """``direct=True``: the file ranges move through libzinf's native I/O engine
    (aio.py: O_DIRECT whole blocks + buffered edges, C worker threads) instead of the
    store's Python workers through the page cache, so the numbers are device bandwidth."""

    def __init__(self, engine, store: TierStore, chunk: int = 4 << 20, slots: int = 3,
                 direct: bool = False, io_threads: int = 8):
        self.e = engine
        self.store = store
        self.chunk = chunk
        self.slots = slots
        self.direct = direct
        dev = engine.dev
        from .store import _PinnedBuffer
        self._bufs = []

        def pinned(n):
            # direct: 4 KiB of slack in front (a range starts at b0 % 4096) and behind
            b = _PinnedBuffer(n * 4 + (8192 if direct else 0))
            self._bufs.append(b)
            return b.tensor if direct else b.tensor.view(torch.float32)
        self.R = [[pinned(chunk) for _ in STATES] for _ in range(slots)]
        self.W = [[pinned(chunk) for _ in STATES] for _ in range(slots)]
        if direct:
            from .aio import AioEngine
            self.aio = AioEngine(io_threads)
        self.S = [[torch.empty(chunk, dtype=torch.float32, device=dev) for _ in STATES]
                  for _ in range(slots)]
        self.ev_h2d = [None] * slots
        self.w_tickets = [[] for _ in range(slots)]
        self.bytes = 0
        self.q: queue.Queue = queue.Queue()
        self.err = None
        self.t = threading.Thread(target=self._run, name="zinf-nvme-opt", daemon=True)
        self.t.start()

    @staticmethod
    def key(bucket: str, state: str, rank: int) -> str:
        return f"{bucket}.{state}/rank{rank}"

    def put_initial(self, bucket: str, rank: int, p32: torch.Tensor) -> None:
        """Write a shard's initial fp32 master and zero moments to NVMe."""
        tk = [self.store.write(self.key(bucket, "p32", rank), p32, TierKind.NVME),
              self.store.write(self.key(bucket, "m", rank), torch.zeros_like(p32), TierKind.NVME),
              self.store.write(self.key(bucket, "v", rank), torch.zeros_like(p32), TierKind.NVME)]
        self.store.flush(tk)

    # -- main-thread side ---------------------------------------------------------
    def submit(self, b, li: int, r: int, contribs, scale: float, ready: torch.cuda.Event,
               p16: torch.Tensor) -> threading.Event:
        done = threading.Event()
        self.q.put((b, li, r, contribs, scale, ready, p16, done))
        return done

    def drain(self) -> None:
        self.q.join()
        if self.err is not None:
            raise self.err

    # -- streamer thread ----------------------------------------------------------
    def _run(self):
        torch.cuda.set_device(self.e.dev)
        while True:
            job = self.q.get()
            if job is None:                        # close(): drop the engine reference
                self.q.task_done()
                self.e = None
                return
            try:
                if self.err is None:
                    self._bucket(*job)
                else:                           # an earlier job failed: release waiters
                    job[-1].ev = None
                    job[-1].set()
            except BaseException as exc:  # noqa: BLE001 — surfaced by drain()
                self.err = exc
                job[-1].ev = None              # no completion event: waiters re-raise err
                job[-1].set()
            finally:
                self.q.task_done()

    def _bucket(self, b, li, r, contribs, scale, ready, p16, done: threading.Event):
        if self.direct:
            return self._bucket_direct(b, li, r, contribs, scale, ready, p16, done)
        e, st, NS = self.e, self.store, self.slots
        L = b.shard
        nch = -(-L // self.chunk)
        cs = -(-L // nch)
        chunks = [(s, min(cs, L - s)) for s in range(0, L, cs)]
        keys = [self.key(b.key, x, r) for x in STATES]
        h2d, opt, d2h = e.h2d_stream, e.opt_stream, e.d2h_stream
        rtk = {}

        def issue_read(ci):
            k = ci % NS
            s, n = chunks[ci]
            if self.ev_h2d[k] is not None:       # R[k]'s previous H2D is done
                self.ev_h2d[k].synchronize()
            rtk[ci] = [st.read_into(keys[j], TierKind.NVME, self.R[k][j][:n], s)
                       for j in range(3)]

        for ci in range(min(NS, len(chunks))):
            issue_read(ci)
        opt.wait_event(ready)
        for ci, (s, n) in enumerate(chunks):
            k = ci % NS
            st.flush(rtk.pop(ci))                 # nc landed in pinned R[k]
            with torch.cuda.stream(h2d):
                for j in range(3):
                    self.S[k][j][:n].copy_(self.R[k][j][:n], non_blocking=True)
                ev_h = torch.cuda.Event()
                ev_h.record(h2d)
            self.ev_h2d[k] = ev_h
            if ci + NS < len(chunks):
                issue_read(ci + NS)
            with torch.cuda.stream(opt):
                opt.wait_event(ev_h)
                sp, sm, sv = (x[:n] for x in self.S[k])
                kernels.rs_adam_dc(contribs, r * L + s, n, b.numel, scale, sp, sm, sv,
                                   p16[s:s + n], e.adam)
                ev_c = torch.cuda.Event()
                ev_c.record(opt)
            st.flush(self.w_tickets[k])           # W[k]'s previous file write is done
            self.w_tickets[k] = []
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_c)
                for j in range(3):
                    self.W[k][j][:n].copy_(self.S[k][j][:n], non_blocking=True)
                ev_d = torch.cuda.Event()
                ev_d.record(d2h)
            ev_d.synchronize()
            self.w_tickets[k] = [st.write_from(keys[j], TierKind.NVME, s, self.W[k][j][:n])
                                 for j in range(3)]
            self.bytes += 2 * 12 * n
        ev_free = torch.cuda.Event()               # contributions no longer read
        ev_free.record(opt)
        done.ev = ev_free
        for k in range(NS):                        # the bucket is durable before the next
            st.flush(self.w_tickets[k])
            self.w_tickets[k] = []
        e.launches += len(chunks)
        done.set()

    def _bucket_direct(self, b, li, r, contribs, scale, ready, p16, done: threading.Event):
        """_bucket over the native I/O engine: file bytes [20 + 4s, 20 + 4(s+n)) of each
        state land at R[k][j] + (b0 % 4096); H2D / D2H use that offset view."""
        from .aio import data_offset
        from .store import SHARD_HEADER_BYTES as HB
        e, NS, aio = self.e, self.slots, self.aio
        L = b.shard
        nch = -(-L // self.chunk)
        cs = -(-L // nch)
        chunks = [(s, min(cs, L - s)) for s in range(0, L, cs)]
        paths = [self.store._nvme_path(self.key(b.key, x, r)) for x in STATES]
        fds = [aio.open(p, write=True) for p in paths]
        h2d, opt, d2h = e.h2d_stream, e.opt_stream, e.d2h_stream
        rids, wids = {}, [[] for _ in range(NS)]

        def rng(s, n):
            b0 = HB + 4 * s
            return b0, b0 + 4 * n, data_offset(b0)

        def view(buf, s, n):
            _, _, d = rng(s, n)
            return buf[d:d + 4 * n].view(torch.float32)

        def issue_read(ci):
            k = ci % NS
            s, n = chunks[ci]
            if self.ev_h2d[k] is not None:       # R[k]'s previous H2D is done
                self.ev_h2d[k].synchronize()
            b0, b1, _ = rng(s, n)
            rids[ci] = [aio.submit(fds[j], False, self.R[k][j].data_ptr(), b0, b1)
                        for j in range(3)]

        try:
            for ci in range(min(NS, len(chunks))):
                issue_read(ci)
            opt.wait_event(ready)
            for ci, (s, n) in enumerate(chunks):
                k = ci % NS
                for rid in rids.pop(ci):          # nc landed in pinned R[k]
                    aio.wait(rid)
                with torch.cuda.stream(h2d):
                    for j in range(3):
                        self.S[k][j][:n].copy_(view(self.R[k][j], s, n), non_blocking=True)
                    ev_h = torch.cuda.Event()
                    ev_h.record(h2d)
                self.ev_h2d[k] = ev_h
                if ci + NS < len(chunks):
                    issue_read(ci + NS)
                with torch.cuda.stream(opt):
                    opt.wait_event(ev_h)
                    sp, sm, sv = (x[:n] for x in self.S[k])
                    kernels.rs_adam_dc(contribs, r * L + s, n, b.numel, scale, sp, sm, sv,
                                       p16[s:s + n], e.adam)
                    ev_c = torch.cuda.Event()
                    ev_c.record(opt)
                for wid in wids[k]:               # W[k]'s previous file write is done
                    aio.wait(wid)
                wids[k] = []
                with torch.cuda.stream(d2h):
                    d2h.wait_event(ev_c)
                    for j in range(3):
                        view(self.W[k][j], s, n).copy_(self.S[k][j][:n], non_blocking=True)
                    ev_d = torch.cuda.Event()
                    ev_d.record(d2h)
                ev_d.synchronize()
                b0, b1, _ = rng(s, n)
                wids[k] = [aio.submit(fds[j], True, self.W[k][j].data_ptr(), b0, b1)
                           for j in range(3)]
                self.bytes += 2 * 12 * n
            ev_free = torch.cuda.Event()          # contributions no longer read
            ev_free.record(opt)
            done.ev = ev_free
            for k in range(NS):                   # the bucket is durable before the next
                for wid in wids[k]:
                    aio.wait(wid)
                wids[k] = []
        finally:
            for ids in list(rids.values()) + wids:
                for rid in ids:
                    try:
                        aio.wait(rid)
                    except OSError:
                        pass
            for f in fds:
                aio.close_file(f)
        self.store._note_nvme_io(24 * L // 2, 24 * L // 2)
        e.launches += len(chunks)
        done.set()

    def close(self):
        """Stop the thread (it holds the engine) and free the pinned slots."""
        if self.t.is_alive():
            self.q.put(None)
            self.t.join()
        self.e = None
        self.S = None
        if getattr(self, "aio", None) is not None:
            self.aio.close()
            self.aio = None
        for b in self._bufs:
            b.free()
        self._bufs = []
