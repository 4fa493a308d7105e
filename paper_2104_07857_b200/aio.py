"""ctypes wrapper of libzinf's native file I/O engine (zi_aio_*, include/zinf.h).

The NVMe tier's direct path ("O_DIRECT into the pinned ring"): worker
threads in C move byte ranges of ``.shard`` files between the disk and pinned host
buffers, whole 4 KiB blocks with O_DIRECT (no page cache) and partial edge blocks through
the page cache. A range [b0, b1) of a file lives at ``buf + b0 % 4096`` in its buffer.
"""

from __future__ import annotations

import ctypes

from . import _lib

BLOCK = 4096


class AioEngine:
    def __init__(self, threads: int = 8):
        self._h = ctypes.c_void_p()
        _lib.call("zi_aio_create", threads, ctypes.byref(self._h))

    def open(self, path: str, write: bool = False, create: bool = False):
        fds = (ctypes.c_int * 2)(-1, -1)
        _lib.call("zi_aio_open", path.encode(), int(write), int(create), fds)
        return fds

    @staticmethod
    def close_file(fds) -> None:
        _lib.call("zi_aio_close", fds)

    def submit(self, fds, write: bool, buf_ptr: int, b0: int, b1: int) -> int:
        rid = ctypes.c_uint64()
        _lib.call("zi_aio_submit", self._h, fds, int(write), buf_ptr, b0, b1, ctypes.byref(rid))
        return rid.value

    def wait(self, rid: int) -> None:
        _lib.call("zi_aio_wait", self._h, rid)

    def close(self) -> None:
        if self._h:
            _lib.call("zi_aio_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass


def data_offset(b0: int) -> int:
    """Where file byte b0 sits in its (4 KiB-aligned) transfer buffer."""
    return b0 % BLOCK
