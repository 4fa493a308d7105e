"""Tensor-level wrappers over the libzinf C ABI.

PyTorch is plumbing here: tensors supply device pointers and the current
CUDA stream; every computation below is a libzinf kernel (csrc/*.cu).
"""

from __future__ import annotations

import torch

from . import _lib

HALF_KIND = {torch.float16: _lib.HALF_FP16, torch.bfloat16: _lib.HALF_BF16}
KIND_DTYPE = {v: k for k, v in HALF_KIND.items()}


def half_kind(dtype: torch.dtype) -> int:
    try:
        return HALF_KIND[dtype]
    except KeyError:
        raise ValueError(f"half dtype must be float16 or bfloat16, got {dtype}") from None


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev(t: torch.Tensor, name: str) -> int:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _dev_or_pinned(t: torch.Tensor, name: str) -> int:
    """Device pointer of a CUDA tensor or of pinned host memory (UVA-addressable)."""
    if t.is_cuda:
        return _dev(t, name)
    if not t.is_contiguous() or not t.is_pinned():
        raise ValueError(f"{name} must be a CUDA tensor or contiguous pinned host memory")
    return t.data_ptr()


def adam_step(p, m, v, g, p_half, consts: _lib.AdamConstsC, stream=None) -> None:
    """zi_adam_step: in-place Adam on fp32 p/m/v with fp32 grad g; p_half <- RNE(p)."""
    n = p.numel()
    for t, nm in ((m, "m"), (v, "v"), (g, "g")):
        if t.numel() != n or t.dtype != torch.float32:
            raise ValueError(f"{nm} must be fp32 with {n} elements")
    if p.dtype != torch.float32:
        raise ValueError("p must be fp32")
    kind = half_kind(p_half.dtype) if p_half is not None else _lib.HALF_BF16
    if p_half is not None and p_half.numel() != n:
        raise ValueError("p_half length mismatch")
    _lib.call("zi_adam_step", _dev(p, "p"), _dev(m, "m"), _dev(v, "v"), _dev(g, "g"),
              _dev(p_half, "p_half") if p_half is not None else None, n, consts, kind,
              _stream(stream))


def _contrib_ptrs(contribs) -> tuple:
    ptrs = []
    for c in contribs:
        if isinstance(c, int):
            ptrs.append(c)          # raw (e.g. IPC-mapped peer) device pointer
        else:
            ptrs.append(_dev(c, "contrib"))
    return _lib.ptr_array(ptrs), len(ptrs)


def reduce_scatter_cast(contribs, shard_offset: int, shard_elems: int, contrib_len: int,
                        scale: float, dtype: torch.dtype, out: torch.Tensor, stream=None) -> None:
    """zi_reduce_scatter_cast: out = scale * fold_k fp32(contribs[k][off:off+n])."""
    if out.dtype != torch.float32 or out.numel() < shard_elems:
        raise ValueError("out must be fp32 with >= shard_elems elements")
    arr, k = _contrib_ptrs(contribs)
    _lib.call("zi_reduce_scatter_cast", arr, k, shard_offset, shard_elems, contrib_len, scale,
              half_kind(dtype), _dev(out, "out"), _stream(stream))


def rs_adam(contribs, shard_offset: int, shard_elems: int, contrib_len: int, scale: float,
            p, m, v, p_half, consts, g_out=None, stream=None) -> None:
    """zi_rs_adam: fused reduce-scatter + cast + scale + Adam + RNE half param."""
    arr, k = _contrib_ptrs(contribs)
    for t, nm in ((p, "p"), (m, "m"), (v, "v")):
        if t.dtype != torch.float32 or t.numel() < shard_elems:
            raise ValueError(f"{nm} must be fp32 with >= shard_elems elements")
    _lib.call("zi_rs_adam", arr, k, shard_offset, shard_elems, contrib_len, scale,
              half_kind(p_half.dtype), _dev(p, "p"), _dev(m, "m"), _dev(v, "v"),
              _dev(p_half, "p_half"), _dev(g_out, "g_out") if g_out is not None else None,
              consts, _stream(stream))


class GraphTimer:
    """A pair of timing events recorded as external nodes (valid inside CUDA graphs)."""

    def __init__(self):
        import ctypes
        self._c = ctypes
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.call("zi_event_create_timed", ctypes.byref(a))
        _lib.call("zi_event_create_timed", ctypes.byref(b))
        self.ev = (a.value, b.value)

    def start(self, stream=None):
        _lib.call("zi_event_record_external", self.ev[0], _stream(stream))

    def stop(self, stream=None):
        _lib.call("zi_event_record_external", self.ev[1], _stream(stream))

    def ms(self) -> float:
        v = self._c.c_float()
        _lib.call("zi_event_elapsed_ms", self.ev[0], self.ev[1], self._c.byref(v))
        return v.value


class DeviceAdamState:
    """Device-resident step counter + folded Adam constants (zi_adam_advance)."""

    def __init__(self, lr: float, betas, eps: float, device="cuda"):
        self.hp = (float(lr), float(betas[0]), float(betas[1]), float(eps))
        self.step = torch.zeros(1, dtype=torch.int32, device=device)
        self.consts = torch.zeros(8, dtype=torch.float32, device=device)

    def advance(self, stream=None) -> None:
        _lib.call("zi_adam_advance", *self.hp, self.step.data_ptr(), self.consts.data_ptr(),
                  _stream(stream))


def rs_adam_dc(contribs, shard_offset: int, shard_elems: int, contrib_len: int, scale: float,
               p, m, v, p_half, state: DeviceAdamState, g_out=None, stream=None) -> None:
    """zi_rs_adam_dc: zi_rs_adam with constants from the device (graph-replayable)."""
    arr, k = _contrib_ptrs(contribs)
    _lib.call("zi_rs_adam_dc", arr, k, shard_offset, shard_elems, contrib_len, scale,
              half_kind(p_half.dtype), _dev(p, "p"), _dev(m, "m"), _dev(v, "v"),
              _dev(p_half, "p_half"), _dev(g_out, "g_out") if g_out is not None else None,
              state.consts.data_ptr(), _stream(stream))


def allgather(shards, shard_elems: int, full: torch.Tensor, full_elems: int,
              use_copy_engine: bool = False, stream=None) -> None:
    """zi_allgather: full[r*L:(r+1)*L] = shards[r], truncated to full_elems."""
    ptrs = [s if isinstance(s, int) else _dev_or_pinned(s, "shard") for s in shards]
    _lib.call("zi_allgather", _lib.ptr_array(ptrs), len(ptrs), shard_elems, full.element_size(),
              _dev(full, "full"), full_elems, int(use_copy_engine), _stream(stream))


def init_uniform(master, p_half, key: int, start_index: int, scale: float, stream=None) -> None:
    n = (master if master is not None else p_half).numel()
    kind = half_kind(p_half.dtype) if p_half is not None else _lib.HALF_BF16
    _lib.call("zi_init_uniform", _dev(master, "master") if master is not None else None,
              _dev(p_half, "p_half") if p_half is not None else None, n, key, start_index,
              scale, kind, _stream(stream))


def fill(master, p_half, value: float, stream=None) -> None:
    n = (master if master is not None else p_half).numel()
    kind = half_kind(p_half.dtype) if p_half is not None else _lib.HALF_BF16
    _lib.call("zi_fill", _dev(master, "master") if master is not None else None,
              _dev(p_half, "p_half") if p_half is not None else None, n, value, kind,
              _stream(stream))


def cast_f32_to_half(src, dst, stream=None) -> None:
    if src.dtype != torch.float32 or dst.numel() != src.numel():
        raise ValueError("cast_f32_to_half: shape/dtype mismatch")
    _lib.call("zi_cast_f32_to_half", _dev(src, "src"), _dev(dst, "dst"), src.numel(),
              half_kind(dst.dtype), _stream(stream))


def cast_half_to_f32(src, dst, stream=None) -> None:
    if dst.dtype != torch.float32 or dst.numel() != src.numel():
        raise ValueError("cast_half_to_f32: shape/dtype mismatch")
    _lib.call("zi_cast_half_to_f32", _dev(src, "src"), _dev(dst, "dst"), src.numel(),
              half_kind(src.dtype), _stream(stream))


def matmul_fixed(a: torch.Tensor, b: torch.Tensor, bias: torch.Tensor | None = None,
                 out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """a @ b (+ bias) for 2-D f32/f64 CUDA views of any strides, summed over k in order
    on one thread per output (zi_matmul_fixed): bit-reproducible, unlike cuBLAS."""
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
        raise ValueError("matmul_fixed: shapes must be (M,K) @ (K,N)")
    if a.dtype not in (torch.float32, torch.float64) or b.dtype != a.dtype:
        raise ValueError("matmul_fixed: f32 or f64 operands of one dtype")
    M, K = a.shape
    N = b.shape[1]
    if out is None:
        out = torch.empty(M, N, dtype=a.dtype, device=a.device)
    if out.shape != (M, N) or out.dtype != a.dtype:
        raise ValueError("matmul_fixed: out shape/dtype mismatch")
    if bias is not None and (bias.dtype != a.dtype or bias.numel() != N or not bias.is_contiguous()):
        raise ValueError("matmul_fixed: bias must be a contiguous (N,) vector of the dtype")
    dt = _lib.DT_F32 if a.dtype == torch.float32 else _lib.DT_F64
    for t, nm in ((a, "a"), (b, "b"), (out, "out")):
        if not t.is_cuda:
            raise ValueError(f"matmul_fixed: {nm} must be a CUDA tensor")
    _lib.call("zi_matmul_fixed", a.data_ptr(), a.stride(0), a.stride(1), b.data_ptr(),
              b.stride(0), b.stride(1), _dev(bias, "bias") if bias is not None else None,
              out.data_ptr(), out.stride(0), out.stride(1), M, N, K, dt, _stream(stream))
    return out


def _operand(t: torch.Tensor, name: str):
    """(pointer, mn_major, ld) of a 2-D bf16 view seen as (rows, k).

    A row-major view (stride(1) == 1) is K-major with ld = stride(0); a
    transposed view (stride(0) == 1) is MN-major with ld = stride(1).
    """
    if t.dtype != torch.bfloat16 or t.dim() != 2 or not t.is_cuda:
        raise ValueError(f"{name}: 2-D bf16 CUDA tensor required")
    if t.stride(1) == 1:
        return t.data_ptr(), 0, t.stride(0)
    if t.stride(0) == 1:
        return t.data_ptr(), 1, t.stride(1)
    raise ValueError(f"{name}: one dimension must be contiguous")


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, bias=None, accumulate=False,
         stream=None) -> torch.Tensor:
    """zi_gemm: out[m, n] (+)= sum_k a[m, k] * b[n, k] (+ bias[n]) on tcgen05.

    ``a`` is (M, K), ``b`` is (N, K); either may be a transposed view
    (MN-major). ``out`` is a row-major bf16 or fp32 (M, N) view.
    """
    M, K = a.shape
    N = b.shape[0]
    if b.shape[1] != K or out.shape != (M, N) or out.stride(1) != 1:
        raise ValueError("gemm: shape mismatch or non-row-major output")
    if out.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("gemm: out must be bf16 or fp32")
    pa, amn, lda = _operand(a, "a")
    pb, bmn, ldb = _operand(b, "b")
    _lib.call("zi_gemm", pa, amn, lda, pb, bmn, ldb,
              _dev(bias, "bias") if bias is not None else None, out.data_ptr(),
              int(out.dtype == torch.float32), int(accumulate), out.stride(0), M, N, K,
              _stream(stream))
    return out


EPI = {"plain": 0, "gelu": 1, "resid": 2, "dgelu": 3, "gelu_save": 4, "mul": 5}


def gemm_ex(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, bias=None, epi: str = "plain",
            x=None, out2=None, stream=None) -> torch.Tensor:
    """zi_gemm_ex: bf16 tcgen05 GEMM with a fused epilogue (see include/zinf.h).

    plain: out = a b^T + bias; gelu: out = u = a b^T + bias, out2 = gelu(u);
    resid: out = (a b^T + bias) + x; dgelu: out = (a b^T) * gelu'(x).
    """
    M, K = a.shape
    N = b.shape[0]
    if b.shape[1] != K or out.shape != (M, N) or out.stride(1) != 1 or out.dtype != torch.bfloat16:
        raise ValueError("gemm_ex: shape mismatch or non-row-major bf16 output")
    for t, name in ((x, "x"), (out2, "out2")):
        if t is not None and (t.shape != (M, N) or t.stride(1) != 1 or t.dtype != torch.bfloat16):
            raise ValueError(f"gemm_ex: {name} must be a row-major bf16 (M, N) view")
    pa, amn, lda = _operand(a, "a")
    pb, bmn, ldb = _operand(b, "b")
    _lib.call("zi_gemm_ex", pa, amn, lda, pb, bmn, ldb,
              _dev(bias, "bias") if bias is not None else None, out.data_ptr(), out.stride(0),
              x.data_ptr() if x is not None else None, x.stride(0) if x is not None else 0,
              out2.data_ptr() if out2 is not None else None,
              out2.stride(0) if out2 is not None else 0, EPI[epi], M, N, K, _stream(stream))
    return out


_SK_WS: dict = {}


def sk_workspace(stream=None) -> torch.Tensor:
    """The stream-K GEMM workspace of (device, stream): flags zeroed once (they reset
    themselves), then one fp32 partial-accumulator slot per CTA. Launches sharing a
    workspace must be stream-ordered, hence one per stream."""
    s = stream if stream is not None else torch.cuda.current_stream()
    key = (s.device.index, s.cuda_stream)
    ws = _SK_WS.get(key)
    if ws is None:
        nbytes = int(_lib.load().zi_gemm_sk_workspace_bytes())
        with torch.cuda.stream(s):
            ws = torch.zeros((nbytes + 255) // 256 * 64, dtype=torch.float32, device=s.device)
        _SK_WS[key] = ws
    return ws


def gemm_sk(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, bias=None, epi: str = "plain",
            x=None, out2=None, split: bool = True, stream=None, colsum=None,
            delta=None, delta_shape=None) -> torch.Tensor:
    """zi_gemm_sk: out = epi(a b^T) on the stream-K tcgen05 GEMM (include/zinf.h).

    ``a`` (M, K) and ``b`` (N, K) as in :func:`gemm` (either may be an MN-major
    transposed view). ``out`` is a row-major bf16 (M, N) view with the epilogues of
    :func:`gemm_ex`, or fp32 (epi "plain", no bias). ``split=False`` runs whole
    tiles (no workspace). Side outputs (zi_gemm_sk_aux): ``colsum`` an fp32
    [ceil(M/32), N] tensor receiving the 32-row block column sums of the bf16 output
    (:func:`colsum_fold` finishes them); ``delta`` an fp32 [B*H*S] tensor receiving
    rowsum(out o x) per (row, head) with ``delta_shape`` = (S, H, D), x = the attention
    output."""
    M, K = a.shape
    N = b.shape[0]
    if b.shape[1] != K or out.shape != (M, N) or out.stride(1) != 1:
        raise ValueError("gemm_sk: shape mismatch or non-row-major output")
    f32 = out.dtype == torch.float32
    if out.dtype not in (torch.bfloat16, torch.float32) or (f32 and (epi != "plain" or bias is not None)):
        raise ValueError("gemm_sk: bf16 output, or fp32 output without an epilogue")
    for t, name in ((x, "x"), (out2, "out2")):
        if t is not None and (t.shape != (M, N) or t.stride(1) != 1 or t.dtype != torch.bfloat16):
            raise ValueError(f"gemm_sk: {name} must be a row-major bf16 (M, N) view")
    pa, amn, lda = _operand(a, "a")
    pb, bmn, ldb = _operand(b, "b")
    s = stream if stream is not None else torch.cuda.current_stream()
    ws = sk_workspace(s) if split else None
    if colsum is not None and (colsum.dtype != torch.float32 or colsum.numel() < -(-M // 32) * N
                               or not colsum.is_contiguous()):
        raise ValueError("gemm_sk: colsum must be contiguous fp32 with ceil(M/32)*N elements")
    dS, dH, dD = delta_shape if delta is not None else (0, 0, 0)
    if delta is not None and (delta.dtype != torch.float32 or delta.numel() != M // max(dS, 1) * dH * dS):
        raise ValueError("gemm_sk: delta must be fp32 [B*H*S]")
    _lib.call("zi_gemm_sk_aux", pa, amn, lda, pb, bmn, ldb,
              _dev(bias, "bias") if bias is not None else None, out.data_ptr(), out.stride(0),
              int(f32), x.data_ptr() if x is not None else None,
              x.stride(0) if x is not None else 0,
              out2.data_ptr() if out2 is not None else None,
              out2.stride(0) if out2 is not None else 0, EPI[epi], M, N, K,
              ws.data_ptr() if ws is not None else None,
              ws.numel() * 4 if ws is not None else 0,
              colsum.data_ptr() if colsum is not None else None,
              delta.data_ptr() if delta is not None else None, dS, dH, dD, s.cuda_stream)
    return out


def colsum_fold(part: torch.Tensor, P: int, N: int, out: torch.Tensor, stream=None) -> None:
    """zi_colsum_fold: out[c] = sum_p part[p, c] in p order (fp32 in; bf16 or fp32 out)."""
    if part.dtype != torch.float32 or part.numel() < P * N or out.numel() != N:
        raise ValueError("colsum_fold: part fp32 [P, N], out [N]")
    _lib.call("zi_colsum_fold", part.data_ptr(), P, N, out.data_ptr(),
              int(out.dtype == torch.float32), _stream(stream))


class Workspace:
    """fp32 scratch for the deterministic column reductions: 1024 self-resetting int
    counters (zeroed here once) followed by per-chunk partial rows. Use one workspace
    per stream: reductions sharing it must be stream-ordered."""

    def __init__(self, elems: int = 8 << 20, device="cuda"):
        self.t = torch.zeros(elems, dtype=torch.float32, device=device)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def __len__(self):
        return self.t.numel()


def _bf16_2d(t: torch.Tensor, name: str):
    if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name}: contiguous bf16 CUDA tensor required")
    return t.data_ptr()


def ln_fwd(x, w, b, y, mean, rstd, eps=1e-5, resid=None, xsum=None, stream=None) -> None:
    """zi_ln_fwd: y = LN(x [+ resid]) * w + b; xsum = x + resid when fused."""
    H = x.shape[-1]
    T = x.numel() // H
    _lib.call("zi_ln_fwd", _bf16_2d(x, "x"), _bf16_2d(resid, "resid") if resid is not None else None,
              _bf16_2d(xsum, "xsum") if xsum is not None else None, _bf16_2d(w, "w"),
              _bf16_2d(b, "b"), _bf16_2d(y, "y"), _dev(mean, "mean"), _dev(rstd, "rstd"), T, H,
              eps, _stream(stream))


def ln_bwd(dy, x, w, mean, rstd, dx, dgamma, dbeta, ws: Workspace, dres=None, dres_sum=None,
           stream=None) -> None:
    """zi_ln_bwd: dx (+ dres), dgamma, dbeta and optionally dres_sum = column sums of
    dres (bf16 or fp32 outputs, all the dtype of dgamma), one pass over the rows."""
    H = x.shape[-1]
    T = x.numel() // H
    f32 = int(dgamma.dtype == torch.float32)
    for g in (dbeta, dres_sum):
        if g is not None and g.dtype != dgamma.dtype:
            raise ValueError("dgamma, dbeta and dres_sum must share a dtype")
    _lib.call("zi_ln_bwd", _bf16_2d(dy, "dy"), _bf16_2d(x, "x"), _bf16_2d(w, "w"),
              _dev(mean, "mean"), _dev(rstd, "rstd"),
              _bf16_2d(dres, "dres") if dres is not None else None, _bf16_2d(dx, "dx"),
              dgamma.data_ptr(), dbeta.data_ptr(),
              dres_sum.data_ptr() if dres_sum is not None else None, f32, ws.ptr, len(ws), T, H,
              _stream(stream))


def gelu_fwd(u, y, stream=None) -> None:
    """zi_gelu_fwd: y = gelu_tanh(u), bf16."""
    if y.shape != u.shape:
        raise ValueError("gelu_fwd: shape mismatch")
    _lib.call("zi_gelu_fwd", _bf16_2d(u, "u"), _bf16_2d(y, "y"), u.numel(), _stream(stream))


def bias_grad(dy, db, ws: Workspace, u=None, du=None, stream=None) -> None:
    """zi_bias_grad: db = column sums of dy; with u: du = gelu'(u) * dy and db = sums of du."""
    N = dy.shape[-1]
    T = dy.numel() // N
    _lib.call("zi_bias_grad", _bf16_2d(dy, "dy"), _bf16_2d(u, "u") if u is not None else None,
              _bf16_2d(du, "du") if du is not None else None, db.data_ptr(),
              int(db.dtype == torch.float32), ws.ptr, len(ws), T, N, _stream(stream))


def softmax_ce(logits, targets, loss_rows, loss, scale: float, stream=None) -> None:
    """zi_softmax_ce: in place (softmax - onehot) * scale; loss_rows and the mean loss."""
    V = logits.shape[-1]
    T = logits.numel() // V
    if targets.dtype != torch.int64 or targets.numel() != T:
        raise ValueError("targets must be int64 with one entry per row")
    _lib.call("zi_softmax_ce", _bf16_2d(logits, "logits"), _dev(targets, "targets"),
              _dev(loss_rows, "loss_rows"), _dev(loss, "loss"), T, V, scale, _stream(stream))


def linear_fwd(x: torch.Tensor, w: torch.Tensor, bias, y: torch.Tensor, stream=None) -> None:
    """zi_linear_fwd (tcgen05 tile GEMM): y = x @ w.T + bias, bf16."""
    M, K = x.shape
    N = w.shape[0]
    if w.shape[1] != K or y.shape != (M, N):
        raise ValueError("linear_fwd: shape mismatch")
    for t in (x, w, y):
        if t.dtype != torch.bfloat16 or t.stride(-1) != 1:
            raise ValueError("linear_fwd: bf16 row-major operands required")
    _lib.call("zi_linear_tile_fwd", x.data_ptr(), w.data_ptr(),
              _dev(bias, "bias") if bias is not None else None, y.data_ptr(), M, K, N,
              x.stride(0), w.stride(0), y.stride(0), _stream(stream))


def linear_tile_bwd(x: torch.Tensor, w_t: torch.Tensor, dy_t: torch.Tensor, dw_t=None,
                    dx_acc=None, db_t=None, stream=None) -> None:
    """zi_linear_tile_bwd: one tile's backward on tcgen05.

    dw_t (bf16 [N_t, K]) = dy_t^T x; dx_acc (fp32 [M, K]) += dy_t w_t;
    db_t (fp32 [N_t]) = column sums of dy_t in a fixed order. ``dy_t`` may be a
    column block of the full upstream gradient (row stride = its width).
    """
    M, K = x.shape
    N = w_t.shape[0]
    if w_t.shape[1] != K or dy_t.shape != (M, N):
        raise ValueError("linear_tile_bwd: shape mismatch")
    for t in (x, w_t, dy_t):
        if t.dtype != torch.bfloat16 or t.stride(-1) != 1 or not t.is_cuda:
            raise ValueError("linear_tile_bwd: bf16 row-major CUDA operands required")
    if dw_t is not None and (dw_t.shape != (N, K) or dw_t.dtype != torch.bfloat16
                             or dw_t.stride(1) != 1):
        raise ValueError("linear_tile_bwd: dw_t must be a row-major bf16 (N_t, K) view")
    if dx_acc is not None and (dx_acc.shape != (M, K) or dx_acc.dtype != torch.float32
                               or dx_acc.stride(1) != 1):
        raise ValueError("linear_tile_bwd: dx_acc must be a row-major fp32 (M, K) view")
    if db_t is not None and (db_t.shape != (N,) or db_t.dtype != torch.float32
                             or not db_t.is_contiguous()):
        raise ValueError("linear_tile_bwd: db_t must be a contiguous fp32 (N_t,) tensor")
    _lib.call("zi_linear_tile_bwd", x.data_ptr(), x.stride(0), w_t.data_ptr(), w_t.stride(0),
              dy_t.data_ptr(), dy_t.stride(0),
              dw_t.data_ptr() if dw_t is not None else None,
              dw_t.stride(0) if dw_t is not None else 0,
              dx_acc.data_ptr() if dx_acc is not None else None,
              dx_acc.stride(0) if dx_acc is not None else 0,
              db_t.data_ptr() if db_t is not None else None, M, K, N, _stream(stream))


def _attn_shapes(qkv: torch.Tensor, batch: int, heads: int):
    if qkv.dtype != torch.bfloat16 or qkv.dim() != 2 or qkv.shape[1] % (3 * heads):
        raise ValueError("qkv must be bf16 [B*S, 3*H*D]")
    if qkv.shape[0] % batch:
        raise ValueError("qkv rows must be batch * seq")
    return qkv.shape[0] // batch, qkv.shape[1] // (3 * heads)


def attn_fwd(qkv: torch.Tensor, out: torch.Tensor, lse: torch.Tensor, batch: int, heads: int,
             stream=None) -> None:
    """zi_attn_fwd: causal attention on tcgen05; out [B*S, H*D] bf16, lse fp32 [B*H*S]
    (log2 domain of the 1/sqrt(D)-scaled scores, kept for the backward)."""
    S, D = _attn_shapes(qkv, batch, heads)
    if out.dtype != torch.bfloat16 or out.shape != (qkv.shape[0], heads * D):
        raise ValueError("out must be bf16 [B*S, H*D]")
    if lse.dtype != torch.float32 or lse.numel() != batch * heads * S:
        raise ValueError("lse must be fp32 with B*H*S elements")
    _lib.call("zi_attn_fwd", _dev(qkv, "qkv"), _dev(out, "out"), _dev(lse, "lse"), batch, heads,
              S, D, _stream(stream))


def attn_bwd(qkv: torch.Tensor, out: torch.Tensor, dout: torch.Tensor, lse: torch.Tensor,
             delta: torch.Tensor, dqkv: torch.Tensor, batch: int, heads: int, stream=None,
             colsum=None) -> None:
    """zi_attn_bwd: dqkv of causal attention, deterministic (fixed-order sums, no
    atomics); delta is an fp32 [B*H*S] workspace (rowsum of dout * out)."""
    S, D = _attn_shapes(qkv, batch, heads)
    for t, nm in ((out, "out"), (dout, "dout")):
        if t is None and nm == "out":   # delta already holds rowsum(dout o out)
            continue
        if t.dtype != torch.bfloat16 or t.shape != (qkv.shape[0], heads * D):
            raise ValueError(f"{nm} must be bf16 [B*S, H*D]")
    if dqkv.dtype != torch.bfloat16 or dqkv.shape != qkv.shape:
        raise ValueError("dqkv must be bf16 like qkv")
    for t, nm in ((lse, "lse"), (delta, "delta")):
        if t.dtype != torch.float32 or t.numel() != batch * heads * S:
            raise ValueError(f"{nm} must be fp32 with B*H*S elements")
    if colsum is not None and (colsum.dtype != torch.float32 or not colsum.is_contiguous()
                               or colsum.numel() < qkv.shape[0] // 32 * qkv.shape[1]):
        raise ValueError("colsum must be contiguous fp32 with B*S/32 * 3*H*D elements")
    _lib.call("zi_attn_bwd_colsum", _dev(qkv, "qkv"),
              _dev(out, "out") if out is not None else None, _dev(dout, "dout"),
              _dev(lse, "lse"), _dev(delta, "delta"), _dev(dqkv, "dqkv"), batch, heads, S, D,
              colsum.data_ptr() if colsum is not None else None, _stream(stream))


def embed_grad(tokens: torch.Tensor, dx: torch.Tensor, acc: torch.Tensor, out: torch.Tensor,
               work: torch.Tensor, stream=None) -> None:
    """zi_embed_grad: out[v] = RNE(acc[v] + sum of dx rows of the tokens with id v, in
    sequence order) — the tied wte gradient without float atomics."""
    T = tokens.numel()
    V, hd = acc.shape
    if tokens.dtype != torch.int64 or dx.shape != (T, hd) or dx.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("tokens int64 [T]; dx bf16 / fp32 [T, hd]")
    if acc.dtype != torch.float32 or out.shape != (V, hd):
        raise ValueError("acc fp32 [V, hd]; out half [V, hd]")
    if work.dtype != torch.int32 or work.numel() < 2 * V + 1 + T:
        raise ValueError("work must be int32 with 2*V + 1 + T elements")
    _lib.call("zi_embed_grad", _dev(tokens.reshape(-1), "tokens"), T, _dev(dx, "dx"),
              int(dx.dtype == torch.float32), _dev(acc, "acc"), V, hd, _dev(out, "out"),
              half_kind(out.dtype), _dev(work, "work"), _stream(stream))


def embed_fwd(tokens: torch.Tensor, wte: torch.Tensor, wpe: torch.Tensor, x: torch.Tensor,
              stream=None) -> None:
    """zi_embed_fwd: x[t] = RNE(wte[tokens[t]] + wpe[t % S]) (bf16; torch's
    F.embedding(tokens, wte) + wpe bit for bit). tokens int64 [B, S] or [T] with S rows of
    wpe; x bf16 [T, hd]."""
    S, hd = wpe.shape
    T = tokens.numel()
    if tokens.dtype != torch.int64 or x.shape != (T, hd) or wte.shape[1] != hd:
        raise ValueError("tokens int64 [T]; wte [V, hd], wpe [S, hd], x [T, hd] bf16")
    _lib.call("zi_embed_fwd", _dev(tokens, "tokens"), T, S, _bf16_2d(wte, "wte"),
              _bf16_2d(wpe, "wpe"), wte.shape[0], hd, _bf16_2d(x, "x"), _stream(stream))


def pos_grad(dx: torch.Tensor, B: int, out: torch.Tensor, stream=None) -> None:
    """zi_pos_grad: out[s] = sum over b ascending of dx[b*S + s] (fp32 sum), stored fp32 or
    rounded RNE to out's half dtype."""
    S, hd = out.shape
    if dx.shape != (B * S, hd) or dx.dtype not in (torch.bfloat16, torch.float16, torch.float32):
        raise ValueError("dx bf16 / fp16 / fp32 [B*S, hd]")
    kind = -1 if out.dtype == torch.float32 else half_kind(out.dtype)
    dkind = -1 if dx.dtype == torch.float32 else half_kind(dx.dtype)
    _lib.call("zi_pos_grad", _dev(dx, "dx"), dkind, B, S, hd,
              _dev(out, "out"), kind, _stream(stream))


def ln_bwd_partials(dy, x, w, mean, rstd, dx, part: torch.Tensor, dres=None, dres_sum=False,
                    stream=None) -> int:
    """zi_ln_bwd_partials: zi_ln_bwd's row pass alone — dx (+ dres), and the CTA partials
    of dgamma, dbeta (and the column sums of dres with dres_sum) as part[sets][P][H].
    Returns P; :func:`fold_sets` folds them (bitwise zi_ln_bwd's gradients)."""
    import ctypes
    H = x.shape[-1]
    T = x.numel() // H
    if part.dtype != torch.float32 or not part.is_cuda:
        raise ValueError("part: fp32 CUDA tensor")
    n = ctypes.c_int(0)
    _lib.call("zi_ln_bwd_partials", _bf16_2d(dy, "dy"), _bf16_2d(x, "x"), _bf16_2d(w, "w"),
              _dev(mean, "mean"), _dev(rstd, "rstd"),
              _bf16_2d(dres, "dres") if dres is not None else None, _bf16_2d(dx, "dx"),
              int(bool(dres_sum)), _dev(part, "part"), part.numel(), T, H, ctypes.byref(n),
              _stream(stream))
    return n.value


def fold_sets(sets, stream=None) -> None:
    """zi_fold_sets: out[c] = sum_p part[p, c] in p order for every (part, P, N, out) set,
    one launch (at most 8 sets; outputs all bf16 or all fp32)."""
    if not 1 <= len(sets) <= _lib.FOLD_MAX_SETS:
        raise ValueError(f"fold_sets: 1..{_lib.FOLD_MAX_SETS} sets")
    f32 = {o.dtype == torch.float32 for _, _, _, o in sets}
    if len(f32) != 1:
        raise ValueError("fold_sets: outputs must share a dtype")
    arr = (_lib.FoldSetC * len(sets))()
    for i, (part, P, N, out) in enumerate(sets):
        if part.dtype != torch.float32 or part.numel() < P * N or out.numel() != N:
            raise ValueError(f"fold_sets: set {i}: part fp32 [P, N], out [N]")
        arr[i] = _lib.FoldSetC(part.data_ptr(), P, N, _dev(out, "out"))
    _lib.call("zi_fold_sets", arr, len(sets), int(f32.pop()), _stream(stream))
