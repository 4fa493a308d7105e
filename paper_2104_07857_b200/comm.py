"""Data-parallel communicators for the partitioned step.

Two implementations of one small interface:

* ``LocalComm(world)`` — ``world`` virtual ranks inside one process on one
  GPU. This is the SPEC's own execution model ("a rank is an index, not an
  OS process") and lets a single B200 run the exact N-rank
  data path: every collective goes through the same libzinf kernels with
  the N shard / gradient buffers as local device pointers.
* ``DistComm()`` — one process per GPU over ``torch.distributed``. Peer
  buffers are exchanged once as CUDA-IPC handles and mapped by the native
  communicator context (``zi_ctx``: rank, world, device, windows), so the
  reduce-scatter and the gather read peer HBM directly over NVLink 5 /
  NVSwitch inside libzinf kernels (or copy engines); ``zi_ctx_barrier``
  orders producers and consumers across GPUs. With the gloo backend and no GPU the host-side plumbing
  (rank layout, handle exchange, object collectives) runs on CPU for tests.
"""

from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib


class _DeviceBuffer:
    """cudaMalloc'd buffer exposed through __cuda_array_interface__ (freed on collection)."""

    _TYPESTR = {torch.float32: "<f4", torch.float16: "<f2", torch.bfloat16: "<V2",
                torch.int32: "<i4", torch.float64: "<f8", torch.uint8: "|u1"}

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _lib.call("zi_device_alloc", max(nbytes, 16), ctypes.byref(p))
        self.ptr = p.value
        self.nbytes = nbytes
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (self.ptr, False), "version": 3}

    def __del__(self):
        try:
            _lib.call("zi_device_free", self.ptr)
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass


def _ipc_tensor(shape, dtype: torch.dtype) -> torch.Tensor:
    n = 1
    for s in shape:
        n *= s
    nbytes = n * torch.empty(0, dtype=dtype).element_size()
    buf = _DeviceBuffer(nbytes)
    t = torch.as_tensor(buf, device="cuda")[:nbytes].view(dtype).view(*shape)
    t.zero_()
    # zeroed before the IPC handle is published: a peer's first write (a barrier
    # arrival) must never be erased by this zero_ landing late on our stream
    torch.cuda.current_stream().synchronize()
    return t


class LocalComm:
    """``world`` simulated ranks in one process."""

    is_local = True

    def __init__(self, world: int = 1):
        if world < 1:
            raise ValueError("world must be >= 1")
        self.world = world
        self.rank = 0  # the process acts for every rank

    def ranks(self):
        return range(self.world)

    def all_ranks_local(self) -> bool:
        return True

    def barrier(self, stream=None) -> None:  # all ranks share one stream order
        return None

    def host_barrier(self) -> None:
        return None

    def allreduce_max(self, x: float) -> float:
        return x

    def alloc(self, shape, dtype: torch.dtype) -> torch.Tensor:
        return torch.zeros(*shape, dtype=dtype, device="cuda")


class DistComm:
    """One process per GPU (torch.distributed); IPC-mapped peer buffers."""

    is_local = False

    def __init__(self, group=None):
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)
        self._chan: dict = {}   # barrier channel -> (flags tensor, its zi_ctx window)
        self._owned: dict[int, int] = {}   # base pointer -> bytes of our shareable buffers
        self._ctx = None        # native zi_ctx (created on first peer-memory use: needs CUDA)
        self.windows: dict[int, int] = {}  # local pointer -> zi_ctx window id
        self._staging: dict = {}  # (name, elems, dtype) -> (shared buffer, peer pointers)
        # barrier flavour: "memop" (stream write / wait-value, no SM held; default) or
        # "kernel" (zi_barrier spin kernel with a device-side epoch)
        self.barrier_kind = os.environ.get("ZI_BARRIER", "memop")
        if self.barrier_kind not in ("memop", "kernel"):
            raise ValueError("ZI_BARRIER must be 'memop' or 'kernel'")
        self._bar_count: dict[int, int] = {}   # channel -> barriers issued (value parity)
        self._capture_mark: dict[int, int] | None = None

    @property
    def ctx(self) -> int:
        """The native communicator context (zi_ctx_create): rank, world, device and
        the IPC-mapped windows; the P2P collectives and barriers run through it."""
        if self._ctx is None:
            c = ctypes.c_void_p()
            _lib.call("zi_ctx_create", self.rank, self.world, torch.cuda.current_device(),
                      ctypes.byref(c))
            self._ctx = c.value
        return self._ctx

    def ranks(self):
        return [self.rank]

    def all_ranks_local(self) -> bool:
        return self.world == 1

    def all_gather_object(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def allreduce_max(self, x: float) -> float:
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    # -- peer memory -------------------------------------------------------------
    def alloc(self, shape, dtype: torch.dtype) -> torch.Tensor:
        """A zeroed CUDA buffer peers can map: its own cudaMalloc (zi_device_alloc),
        so the IPC handle names exactly this buffer."""
        _ = self.ctx            # zi_ctx_create pins libzinf's device to this rank's GPU
        t = _ipc_tensor(shape, dtype)
        self._owned[t.data_ptr()] = t.untyped_storage().nbytes()
        return t

    def share(self, t: torch.Tensor) -> list[int]:
        """Device pointers of every rank's copy of a same-shaped buffer (IPC).

        Collective: every rank calls it with a view of a buffer from ``alloc``.
        Returns our own pointer at index ``rank`` and IPC mappings of the
        peers' buffers (same offset) elsewhere.
        """
        if not t.is_cuda:
            raise ValueError("share() needs a CUDA tensor")
        ptr = t.data_ptr()
        base = next((b for b, n in self._owned.items() if b <= ptr < b + n), None)
        if base is None:
            raise ValueError("share() needs a view of a DistComm.alloc() buffer")
        h = (ctypes.c_char * 64)()
        _lib.call("zi_ipc_get_handle", base, h)
        infos = self.all_gather_object((bytes(h), ptr - base))
        handles = b"".join(hb for hb, _ in infos)
        offs = (ctypes.c_uint64 * self.world)(*[off for _, off in infos])
        win = ctypes.c_int()
        # zi_ctx maps each peer allocation once (lazy peer access over NVLink)
        _lib.call("zi_ctx_add_window", self.ctx, ptr, handles, offs, ctypes.byref(win))
        arr = (ctypes.c_void_p * self.world)()
        _lib.call("zi_ctx_window_ptrs", self.ctx, win.value, arr)
        self.windows[ptr] = win.value
        return [int(a) for a in arr]

    def window(self, t: torch.Tensor) -> int:
        """zi_ctx window id of a buffer passed to ``share``."""
        return self.windows[t.data_ptr()]

    def allgather_window(self, t: torch.Tensor, shard_elems: int, full: torch.Tensor,
                         offset_elems: int = 0, use_copy_engine: bool = False,
                         stream=None) -> None:
        """SPEC allgather over a shared window (zi_ctx_allgather): full = concat over
        ranks of window_r[offset : offset + shard], truncated to full.numel()."""
        dt = {torch.float32: _lib.DT_F32, torch.float64: _lib.DT_F64,
              torch.float16: _lib.DT_F16, torch.bfloat16: _lib.DT_BF16}[t.dtype]
        s = stream if stream is not None else torch.cuda.current_stream()
        _lib.call("zi_ctx_allgather", self.ctx, self.window(t), offset_elems * t.element_size(),
                  shard_elems, dt, full.data_ptr(), full.numel(), int(use_copy_engine),
                  s.cuda_stream)

    def reduce_scatter_window(self, t: torch.Tensor, shard_elems: int, out: torch.Tensor,
                              scale: float, contrib_len: int | None = None,
                              offset_elems: int = 0, stream=None) -> None:
        """SPEC reduce_scatter + cast over a shared half window (zi_ctx_reduce_scatter_cast):
        out (fp32, our shard) = scale * rank-order fold of every rank's bucket."""
        from .kernels import half_kind
        s = stream if stream is not None else torch.cuda.current_stream()
        n = t.numel() - offset_elems if contrib_len is None else contrib_len
        _lib.call("zi_ctx_reduce_scatter_cast", self.ctx, self.window(t),
                  offset_elems * t.element_size(), n, shard_elems, scale, half_kind(t.dtype),
                  out.data_ptr(), s.cuda_stream)

    def staging(self, name: str, elems: int, dtype: torch.dtype) -> tuple[torch.Tensor, list[int]]:
        """A persistent shared window of ``elems`` (allocated and IPC-mapped once per name).

        Collective on first use. The SPEC collectives over tier-store shards
        (partition.allgather / reduce_scatter with a DistComm) copy the local
        shard in, so one window per PartitionedTensor serves every call and
        the zi_ctx window table does not grow per call.
        """
        k = (name, int(elems), dtype)
        if k not in self._staging:
            t = self.alloc((max(1, int(elems)),), dtype)
            self._staging[k] = (t, self.share(t))
        return self._staging[k]

    def open_channels(self, channels=(0, 1, 2)) -> None:
        """Create barrier channels eagerly (collective), then a host barrier, so no
        channel's flag window is created lazily in the middle of a step on a
        stream that is not ordered after its zeroing."""
        if self.world == 1:
            return
        for ch in channels:
            self._channel(ch)
        self.host_barrier()

    def _channel(self, channel: int):
        if channel not in self._chan:   # collective on first use of the channel
            flags = self.alloc((2 * self.world,), torch.int32)   # two slot sets
            self.share(flags)
            self._chan[channel] = (flags, self.window(flags))
        return self._chan[channel]

    def device_barrier(self, stream=None, channel: int = 0) -> None:
        """zi_barrier over IPC flag words (orders P2P reads with peer writers).

        Each channel has its own flag array and epoch counter: barriers issued
        on different CUDA streams (compute vs gather) must not share one, or
        an epoch reached on one stream would release waiters on the other.
        Every rank must issue the barriers of a channel in the same order.
        """
        if self.world == 1:
            return
        win = self._channel(channel)[1]
        s = stream if stream is not None else torch.cuda.current_stream()
        if self.barrier_kind == "kernel":
            _lib.call("zi_ctx_barrier", self.ctx, win, s.cuda_stream)
            return
        n = self._bar_count.get(channel, 0)
        self._bar_count[channel] = n + 1
        _lib.call("zi_ctx_barrier_value", self.ctx, win, n % 2, s.cuda_stream)

    def begin_capture(self) -> None:
        """Mark the barrier counts before a CUDA-graph capture (see end_capture)."""
        self._capture_mark = dict(self._bar_count)

    def end_capture(self, stream=None) -> None:
        """Before the capture ends: pad every channel whose captured barrier count is
        odd with one more barrier, so each replay leaves the slot-set parity where it
        found it and replays / eager calls keep alternating (zi_ctx_barrier_value)."""
        mark, self._capture_mark = self._capture_mark or {}, None
        if self.barrier_kind != "memop":
            return
        for ch, n in sorted(self._bar_count.items()):
            if (n - mark.get(ch, 0)) % 2:
                self.device_barrier(stream, channel=ch)

    def host_barrier(self) -> None:
        """Every rank's host reached this point (torch.distributed barrier)."""
        dist.barrier(group=self.group)

    def barrier(self, stream=None) -> None:
        if self.backend == "nccl":
            self.device_barrier(stream)
        else:
            dist.barrier(group=self.group)

    def close(self) -> None:
        """zi_ctx_destroy: unmaps every peer window (peers must be done reading ours)."""
        if self._ctx is not None:
            _lib.call("zi_ctx_destroy", self._ctx)
            self._ctx = None
            self.windows.clear()
            self._chan.clear()
            self._staging.clear()
