"""tcgen05 tile GEMM (zi_linear_fwd) against an fp32 torch reference.

Tolerance: the kernel accumulates in fp32 and rounds once to bf16, so the
result must lie within 1 bf16 ulp (2^-7 relative) of the fp32 reference
plus a small absolute term for accumulation-order differences.
"""

import pytest
import torch

from paper_2104_07857_b200 import kernels

pytestmark = pytest.mark.gpu


def ref(x, w, b):
    y = x.float() @ w.float().t()
    if b is not None:
        y = y + b.float()
    return y


def check(y, yr, K):
    # one bf16 ulp (2^-7 relative): RNE is half an ulp, and fp32 accumulation-order
    # differences vs the reference can move a value across a rounding boundary
    # plus K * 2^-20 absolute: fp32 sums of K O(1) products in a different order
    # differ by ~K * eps32 where the result cancels to near zero
    err = (y.float() - yr).abs()
    tol = yr.abs() * 2 ** -7 + K * 2 ** -20
    bad = (err > tol).sum().item()
    assert bad == 0, f"{bad} elements out of tolerance; max err {err.max().item()}"


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 1024), (300, 520, 200),
                                   (1, 8, 8), (1000, 4104, 4096), (2048, 2048, 16384)])
@pytest.mark.parametrize("bias", [False, True])
def test_linear_fwd(M, N, K, bias):
    torch.manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * K ** -0.5
    b = torch.randn(N, device="cuda", dtype=torch.bfloat16) if bias else None
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    kernels.linear_fwd(x, w, b, y)
    torch.cuda.synchronize()
    check(y, ref(x, w, b), K)


@pytest.mark.parametrize("T,din,dout", [(256, 512, 1024), (1000, 320, 200), (8192, 2048, 6144)])
@pytest.mark.parametrize("f32", [False, True])
def test_backward_gemms(T, din, dout, f32):
    """dx = dy W (B N-major) and dW = dy^T x (A and B MN-major) on tcgen05."""
    torch.manual_seed(T + din)
    x = torch.randn(T, din, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(dout, din, device="cuda", dtype=torch.bfloat16) * din ** -0.5
    dy = torch.randn(T, dout, device="cuda", dtype=torch.bfloat16)
    odt = torch.float32 if f32 else torch.bfloat16
    dx = torch.empty(T, din, device="cuda", dtype=odt)
    kernels.gemm(dy, w.t(), dx)
    dW = torch.empty(dout, din, device="cuda", dtype=odt)
    kernels.gemm(dy.t(), x.t(), dW)
    torch.cuda.synchronize()
    check(dx, dy.float() @ w.float(), dout)
    check(dW, dy.float().t() @ x.float(), T)


def test_accumulate_fp32():
    """dx += g_t W_t over tiles (backward_tiled's running sum) in fp32."""
    torch.manual_seed(0)
    T, din, dout = 512, 768, 1024
    g = torch.randn(T, dout, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(dout, din, device="cuda", dtype=torch.bfloat16) * din ** -0.5
    acc = torch.zeros(T, din, device="cuda", dtype=torch.float32)
    for s in range(0, dout, 256):
        kernels.gemm(g[:, s:s + 256], w[s:s + 256].t(), acc, accumulate=True)
    torch.cuda.synchronize()
    ref = g.float() @ w.float()
    assert ((acc - ref).abs() <= 1e-3 * (1 + ref.abs())).all()


def test_linear_fwd_strided_views():
    """Tiles of a larger weight / output (ld > row length), as forward_tiled uses them."""
    M, K, Nfull, T = 256, 512, 1024, 4
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(Nfull, K, device="cuda", dtype=torch.bfloat16) * K ** -0.5
    y = torch.zeros(M, Nfull, device="cuda", dtype=torch.bfloat16)
    R = Nfull // T
    for t in range(T):
        kernels.linear_fwd(x, w[t * R:(t + 1) * R], None, y[:, t * R:(t + 1) * R])
    torch.cuda.synchronize()
    check(y, ref(x, w, None), K)


@pytest.mark.parametrize("wide", ["0", "1"])
@pytest.mark.parametrize("M,N,K", [(256, 512, 128), (1000, 1032, 320), (2048, 6144, 2048),
                                   (520, 2048, 8192)])
@pytest.mark.parametrize("layout", ["fwd", "dx", "dw"])
def test_wide_and_narrow_tiles(M, N, K, layout, wide):
    """gemm_ex (always the 256x512 pair tile) and gemm (heuristic) on every operand layout."""
    torch.manual_seed(M * 7 + N + K)
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * K ** -0.5
    if layout == "dx":     # B N-major: b is a transposed view of a (K, N) tensor
        b = b.t().contiguous().t()
    if layout == "dw":     # A and B MN-major
        a = a.t().contiguous().t()
        b = b.t().contiguous().t()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    kernels.gemm_ex(a, b, y) if wide == "1" else kernels.gemm(a, b, y)
    torch.cuda.synchronize()
    check(y, a.float() @ b.float().t(), K)


@pytest.mark.parametrize("M,N,K", [(8192, 8192, 2048), (300, 1032, 256), (1024, 2048, 8192)])
@pytest.mark.parametrize("epi", ["bias", "gelu", "resid", "dgelu"])
def test_fused_epilogues(M, N, K, epi):
    """Each fused epilogue against the unfused bf16 sequence of torch ops."""
    import torch.nn.functional as F
    torch.manual_seed(M + N)
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * K ** -0.5
    bias = torch.randn(N, device="cuda", dtype=torch.bfloat16)
    acc = x.float() @ w.float().t()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    if epi == "bias":
        kernels.gemm_ex(x, w, out, bias=bias)
        check(out, acc + bias.float(), K)
    elif epi == "gelu":
        g = torch.empty_like(out)
        kernels.gemm_ex(x, w, out, bias=bias, epi="gelu", out2=g)
        check(out, acc + bias.float(), K)
        gr = F.gelu(out.float(), approximate="tanh")
        err = (g.float() - gr).abs()
        assert (err <= gr.abs() * 2 ** -7 + 2e-3).all(), err.max().item()
    elif epi == "resid":
        r = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
        kernels.gemm_ex(x, w, out, bias=bias, epi="resid", x=r)
        y = acc + bias.float()
        ref = y.bfloat16().float() + r.float()
        # two roundings as in the unfused path: bf16(y) then bf16(bf16(y) + r); the
        # first can move by one ulp of |y| (fp32 accumulation order), which is not
        # small relative to ref when y and r cancel
        err = (out.float() - ref).abs()
        tol = ref.abs() * 2 ** -7 + y.abs() * 2 ** -7 + K * 2 ** -20
        assert (err <= tol).all(), err.max().item()
    else:
        u = (acc + bias.float()).bfloat16()
        kernels.gemm_ex(x, w, out, epi="dgelu", x=u)
        dref = torch.ops.aten.gelu_backward(acc.bfloat16().float(), u.float(), approximate="tanh")
        err = (out.float() - dref).abs()
        assert (err <= dref.abs() * 2 ** -6 + K * 2 ** -19 + 2e-3).all(), err.max().item()


@pytest.mark.gpu
@pytest.mark.parametrize("M,K,N_t,width", [(256, 128, 192, 384), (300, 256, 136, 200)])
def test_linear_tile_bwd(M, K, N_t, width):
    """zi_linear_tile_bwd on a column block of the upstream grad (the tiled backward's
    access pattern) against fp32 torch: dW_t, dx accumulate, db_t (fixed-order sums)."""
    torch.manual_seed(1)
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N_t, K, device="cuda").bfloat16()
    gy = torch.randn(M, width, device="cuda").bfloat16()
    s0 = width - N_t
    g = gy[:, s0:]
    dw = torch.empty(N_t, K, device="cuda", dtype=torch.bfloat16)
    dx0 = torch.randn(M, K, device="cuda")
    dx = dx0.clone()
    db = torch.empty(N_t, device="cuda")
    kernels.linear_tile_bwd(x, w, g, dw_t=dw, dx_acc=dx, db_t=db)
    db2 = torch.empty_like(db)
    kernels.linear_tile_bwd(x, w, g, db_t=db2)
    torch.cuda.synchronize()
    gf, xf, wf = g.float(), x.float(), w.float()
    torch.testing.assert_close(dw.float(), gf.t() @ xf, rtol=1e-2, atol=1e-2 * M ** 0.5)
    torch.testing.assert_close(dx, dx0 + gf @ wf, rtol=1e-3, atol=1e-3 * N_t ** 0.5)
    torch.testing.assert_close(db, gf.sum(0), rtol=1e-5, atol=1e-4)
    assert torch.equal(db, db2)    # deterministic


@pytest.mark.gpu
def test_h2d_d2h_async_with_event():
    from paper_2104_07857_b200 import _lib
    from paper_2104_07857_b200 import store as S
    import ctypes
    pool = S.BufferPool(1 << 20, 2, pinned=True)
    a, b = pool.acquire(), pool.acquire()
    S._buf_tensor(a)[:] = torch.randint(0, 255, (1 << 20,), dtype=torch.uint8)
    d = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    ev = ctypes.c_void_p()
    _lib.call("zi_event_create", ctypes.byref(ev))
    s = torch.cuda.Stream()
    _lib.call("zi_h2d_async", d.data_ptr(), a.ptr, 1 << 20, s.cuda_stream, ev)
    _lib.call("zi_d2h_async", b.ptr, d.data_ptr(), 1 << 20, s.cuda_stream, ev)
    _lib.call("zi_event_sync", ev)
    assert torch.equal(S._buf_tensor(a), S._buf_tensor(b))
    _lib.call("zi_event_destroy", ev)
    pool.release(a)
    pool.release(b)
