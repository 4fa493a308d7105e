"""ctypes binding of libzinf.so (include/zinf.h).

The product path has no fallback: if the shared library is missing or a
call fails, an exception is raised. Status codes map onto the reference
exception tree (store.py:54-71) through ``check``.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libzinf.so")

ZI_OK, ZI_EINVAL, ZI_ECAPACITY, ZI_ENOTFOUND, ZI_ECUDA, ZI_ENCCL, ZI_EEXHAUSTED, ZI_EIO = range(8)
HALF_FP16, HALF_BF16 = 0, 1
DT_F32, DT_F16, DT_F64, DT_BF16 = 0, 1, 2, 3

c_void_p = ctypes.c_void_p
c_size_t = ctypes.c_size_t
c_int = ctypes.c_int
c_float = ctypes.c_float
c_uint64 = ctypes.c_uint64
c_uint32 = ctypes.c_uint32


class AdamConstsC(ctypes.Structure):
    _fields_ = [(n, c_float) for n in ("lr", "b1", "omb1", "b2", "omb2", "bc1", "bc2", "eps")]


# name -> argtypes (restype is always int unless listed in _RESTYPE)
SIGNATURES = {
    "zi_last_error": [],
    "zi_version": [],
    "zi_adam_step": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                     ctypes.POINTER(AdamConstsC), c_int, c_void_p],
    "zi_reduce_scatter_cast": [ctypes.POINTER(c_void_p), c_int, c_size_t, c_size_t, c_size_t,
                               c_float, c_int, c_void_p, c_void_p],
    "zi_reduce_scatter": [ctypes.POINTER(c_void_p), c_int, c_size_t, c_size_t, c_size_t, c_int,
                          ctypes.c_double, c_void_p, c_void_p],
    "zi_rs_adam": [ctypes.POINTER(c_void_p), c_int, c_size_t, c_size_t, c_size_t, c_float, c_int,
                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                   ctypes.POINTER(AdamConstsC), c_void_p],
    "zi_rs_adam_dc": [ctypes.POINTER(c_void_p), c_int, c_size_t, c_size_t, c_size_t, c_float,
                      c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "zi_adam_advance": [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                        c_void_p, c_void_p, c_void_p],
    "zi_allgather": [ctypes.POINTER(c_void_p), c_int, c_size_t, c_size_t, c_void_p, c_size_t,
                     c_int, c_void_p],
    "zi_barrier": [ctypes.POINTER(c_void_p), c_int, c_int, c_uint32, c_void_p],
    "zi_barrier_dev": [ctypes.POINTER(c_void_p), c_int, c_int, c_void_p, c_void_p],
    "zi_init_uniform": [c_void_p, c_void_p, c_size_t, c_uint64, c_uint64, c_float, c_int, c_void_p],
    "zi_fill": [c_void_p, c_void_p, c_size_t, c_float, c_int, c_void_p],
    "zi_cast_f32_to_half": [c_void_p, c_void_p, c_size_t, c_int, c_void_p],
    "zi_cast_half_to_f32": [c_void_p, c_void_p, c_size_t, c_int, c_void_p],
    "zi_matmul_fixed": [c_void_p, ctypes.c_int64, ctypes.c_int64, c_void_p, ctypes.c_int64,
                        ctypes.c_int64, c_void_p, c_void_p, ctypes.c_int64, ctypes.c_int64, c_int,
                        c_int, c_int, c_int, c_void_p],
    "zi_ln_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                  c_int, c_int, c_float, c_void_p],
    "zi_ln_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                  c_void_p, c_void_p, c_int, c_void_p, c_size_t, c_int, c_int, c_void_p],
    "zi_gelu_fwd": [c_void_p, c_void_p, c_size_t, c_void_p],
    "zi_bias_grad": [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_size_t, c_int,
                     c_int, c_void_p],
    "zi_softmax_ce": [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_float, c_void_p],
    "zi_host_alloc": [c_size_t, ctypes.POINTER(c_void_p)],
    "zi_host_free": [c_void_p],
    "zi_memcpy_async": [c_void_p, c_void_p, c_size_t, c_int, c_void_p],
    "zi_event_create": [ctypes.POINTER(c_void_p)],
    "zi_event_destroy": [c_void_p],
    "zi_event_create_timed": [ctypes.POINTER(c_void_p)],
    "zi_event_record_external": [c_void_p, c_void_p],
    "zi_event_elapsed_ms": [c_void_p, c_void_p, ctypes.POINTER(c_float)],
    "zi_event_record": [c_void_p, c_void_p],
    "zi_event_query": [c_void_p],
    "zi_event_sync": [c_void_p],
    "zi_stream_wait_event": [c_void_p, c_void_p],
    "zi_pool_create": [c_size_t, c_int, c_int, c_int, ctypes.POINTER(c_void_p)],
    "zi_pool_destroy": [c_void_p],
    "zi_pool_buffer": [c_void_p, c_int, ctypes.POINTER(c_void_p)],
    "zi_pool_acquire": [c_void_p, ctypes.POINTER(c_int)],
    "zi_pool_release": [c_void_p, c_int],
    "zi_pool_stats": [c_void_p, ctypes.POINTER(c_int), ctypes.POINTER(c_uint64)],
    "zi_h2d_async": [c_void_p, c_void_p, c_size_t, c_void_p, c_void_p],
    "zi_d2h_async": [c_void_p, c_void_p, c_size_t, c_void_p, c_void_p],
    "zi_linear_tile_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                           c_int, c_int, c_void_p],
    "zi_linear_tile_bwd": [c_void_p, c_int, c_void_p, c_int, c_void_p, c_int, c_void_p, c_int,
                           c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_void_p],
    "zi_aio_create": [c_int, ctypes.POINTER(c_void_p)],
    "zi_aio_destroy": [c_void_p],
    "zi_aio_open": [ctypes.c_char_p, c_int, c_int, ctypes.POINTER(c_int)],
    "zi_aio_close": [ctypes.POINTER(c_int)],
    "zi_aio_truncate": [ctypes.POINTER(c_int), c_size_t],
    "zi_aio_submit": [c_void_p, ctypes.POINTER(c_int), c_int, c_void_p, c_size_t, c_size_t,
                      ctypes.POINTER(c_uint64)],
    "zi_aio_wait": [c_void_p, c_uint64],
    "zi_device_alloc": [c_size_t, ctypes.POINTER(c_void_p)],
    "zi_device_free": [c_void_p],
    "zi_ipc_get_handle": [c_void_p, ctypes.c_char_p],
    "zi_ipc_open": [ctypes.c_char_p, ctypes.POINTER(c_void_p)],
    "zi_ipc_close": [c_void_p],
    "zi_ctx_create": [c_int, c_int, c_int, ctypes.POINTER(c_void_p)],
    "zi_ctx_destroy": [c_void_p],
    "zi_ctx_info": [c_void_p, ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int)],
    "zi_ctx_add_window": [c_void_p, c_void_p, ctypes.c_char_p, ctypes.POINTER(c_uint64),
                          ctypes.POINTER(c_int)],
    "zi_ctx_window_ptrs": [c_void_p, c_int, ctypes.POINTER(c_void_p)],
    "zi_ctx_allgather": [c_void_p, c_int, c_size_t, c_size_t, c_int, c_void_p, c_size_t, c_int,
                         c_void_p],
    "zi_ctx_reduce_scatter_cast": [c_void_p, c_int, c_size_t, c_size_t, c_size_t, c_float, c_int,
                                   c_void_p, c_void_p],
    "zi_ctx_barrier": [c_void_p, c_int, c_void_p],
    "zi_ctx_barrier_value": [c_void_p, c_int, c_int, c_void_p],
    "zi_linear_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int,
                      c_int, c_void_p],
    "zi_gemm": [c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_void_p, c_void_p, c_int, c_int,
                c_int, c_int, c_int, c_int, c_void_p],
    "zi_gemm_set_profile": [c_void_p],
    "zi_attn_set_trace": [c_void_p],
    "zi_embed_grad": [c_void_p, c_int, c_void_p, c_int, c_void_p, c_int, c_int, c_void_p, c_int,
                      c_void_p, c_void_p],
    "zi_ln_bwd_partials": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                           c_int, c_void_p, c_size_t, c_int, c_int, c_void_p, c_void_p],
    "zi_fold_sets": [c_void_p, c_int, c_int, c_void_p],
    "zi_embed_fwd": [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p],
    "zi_pos_grad": [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int, c_void_p],
    "zi_attn_fwd": [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p],
    "zi_attn_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                    c_int, c_void_p],
    "zi_gemm_ex": [c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_void_p, c_void_p, c_int,
                   c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p],
    "zi_gemm_sk": [c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_void_p, c_void_p, c_int,
                   c_int, c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p,
                   c_size_t, c_void_p],
    "zi_gemm_sk_aux": [c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_void_p, c_void_p, c_int,
                       c_int, c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int, c_int,
                       c_void_p, c_size_t, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p],
    "zi_colsum_fold": [c_void_p, c_int, c_int, c_void_p, c_int, c_void_p],
    "zi_attn_bwd_colsum": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                           c_int, c_int, c_int, c_void_p, c_void_p],
    "zi_gemm_sk_workspace_bytes": [],
    "zi_launch_count": [],
}
_RESTYPE = {"zi_last_error": ctypes.c_char_p, "zi_gemm_sk_workspace_bytes": c_size_t,
            "zi_launch_count": ctypes.c_longlong}

_lib = None
_lock = threading.Lock()


class ZinfError(RuntimeError):
    """A libzinf call failed (CUDA / NCCL / argument error)."""


def load() -> ctypes.CDLL:
    """Load libzinf.so once; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ZinfError(f"{LIB_PATH} not found: build it with `make` or "
                                "`python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = _RESTYPE.get(name, c_int)
            _lib = L
    return _lib


def last_error() -> str:
    return load().zi_last_error().decode(errors="replace")


def check(status: int, what: str) -> None:
    if status == ZI_OK:
        return
    msg = f"{what}: {last_error()}"
    from .store import CapacityExceeded, KeyNotFound, PoolExhausted  # late: no cycle at load
    if status == ZI_EEXHAUSTED:
        raise PoolExhausted(msg)
    if status == ZI_EIO:
        raise OSError(msg)
    if status == ZI_ECAPACITY:
        raise CapacityExceeded(msg)
    if status == ZI_ENOTFOUND:
        raise KeyNotFound(msg)
    if status == ZI_EINVAL:
        raise ValueError(msg)
    raise ZinfError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


class FoldSetC(ctypes.Structure):
    """include/zinf.h zi_fold_set."""
    _fields_ = [("part", c_void_p), ("P", c_int), ("N", c_int), ("out", c_void_p)]


FOLD_MAX_SETS = 8


def ptr_array(ptrs) -> "ctypes.Array":
    arr = (c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = int(p)
    return arr


def adam_consts(lr: float, beta1: float, beta2: float, eps: float, step: int) -> AdamConstsC:
    """Host constant folding identical to oracle/adam.py AdamConsts.make.

    Python doubles rounded once to float32 by ctypes (IEEE RNE), as numpy's
    np.float32(...) does.
    """
    if step < 1:
        raise ValueError("Adam step counter starts at 1")
    return AdamConstsC(lr, beta1, 1.0 - beta1, beta2, 1.0 - beta2,
                       1.0 - beta1 ** step, 1.0 - beta2 ** step, eps)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def launch_count() -> int:
    """Kernels libzinf has launched in this process (zi_launch_count)."""
    return int(load().zi_launch_count())
