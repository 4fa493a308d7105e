"""Fused block kernels (csrc/fused.cu) against plain fp32 PyTorch references.

Tolerances: outputs are bf16, so 2^-7 relative (one bf16 ulp) plus an
absolute term scaled by the reduction length; column reductions are
additionally checked for determinism (bit-identical on re-run).
"""

import pytest
import torch
import torch.nn.functional as F

from paper_2104_07857_b200 import kernels as K

pytestmark = pytest.mark.gpu


def close(a, b, rtol=2 ** -7, atol=1e-2):
    a, b = a.float(), b.float()
    bad = ((a - b).abs() > rtol * b.abs() + atol).sum().item()
    assert bad == 0, f"{bad} mismatches, max err {(a - b).abs().max().item()}"


@pytest.mark.parametrize("T,H", [(64, 128), (1000, 256), (8192, 2048), (513, 1024), (300, 4096),
                                 (257, 8192)])
@pytest.mark.parametrize("resid", [False, True])
def test_ln_fwd(T, H, resid):
    g = torch.Generator(device="cuda").manual_seed(T + H)
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    r = torch.randn(T, H, device="cuda", generator=g).bfloat16() if resid else None
    w = (1 + 0.1 * torch.randn(H, device="cuda", generator=g)).bfloat16()
    b = (0.1 * torch.randn(H, device="cuda", generator=g)).bfloat16()
    y = torch.empty_like(x)
    xs = torch.empty_like(x) if resid else None
    mean = torch.empty(T, device="cuda")
    rstd = torch.empty(T, device="cuda")
    K.ln_fwd(x, w, b, y, mean, rstd, resid=r, xsum=xs)
    xin = (x.float() + r.float()).bfloat16() if resid else x
    if resid:
        assert torch.equal(xs, xin)
    ref = F.layer_norm(xin.float(), (H,), w.float(), b.float(), 1e-5)
    close(y, ref)
    torch.testing.assert_close(mean, xin.float().mean(-1), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("T,H", [(64, 128), (1000, 256), (8192, 2048), (300, 4096), (257, 8192)])
@pytest.mark.parametrize("dres", [False, True])
def test_ln_bwd(T, H, dres):
    g = torch.Generator(device="cuda").manual_seed(T * H)
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    w = (1 + 0.1 * torch.randn(H, device="cuda", generator=g)).bfloat16()
    b = torch.zeros(H, device="cuda").bfloat16()
    dy = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    dr = torch.randn(T, H, device="cuda", generator=g).bfloat16() if dres else None
    y = torch.empty_like(x)
    mean = torch.empty(T, device="cuda")
    rstd = torch.empty(T, device="cuda")
    K.ln_fwd(x, w, b, y, mean, rstd)
    dx = torch.empty_like(x)
    dg = torch.empty(H, device="cuda", dtype=torch.float32)
    db = torch.empty(H, device="cuda", dtype=torch.float32)
    ds = torch.empty(H, device="cuda", dtype=torch.float32) if dres else None
    ws = K.Workspace()
    K.ln_bwd(dy, x, w, mean, rstd, dx, dg, db, ws, dres=dr, dres_sum=ds)
    xr = x.float().requires_grad_(True)
    wr = w.float().requires_grad_(True)
    br = b.float().requires_grad_(True)
    F.layer_norm(xr, (H,), wr, br, 1e-5).backward(dy.float())
    ref_dx = xr.grad + (dr.float() if dres else 0)
    close(dx, ref_dx, atol=2e-2)
    torch.testing.assert_close(dg, wr.grad, rtol=1e-3, atol=1e-3 * T ** 0.5)
    torch.testing.assert_close(db, br.grad, rtol=1e-3, atol=1e-3 * T ** 0.5)
    if dres:   # the fused bias gradient of the linear that produced dres
        torch.testing.assert_close(ds, dr.float().sum(0), rtol=1e-3, atol=1e-3 * T ** 0.5)
    dg2 = torch.empty_like(dg)
    db2 = torch.empty_like(db)
    K.ln_bwd(dy, x, w, mean, rstd, dx, dg2, db2, ws, dres=dr)
    assert torch.equal(dg, dg2) and torch.equal(db, db2)   # deterministic


@pytest.mark.parametrize("n", [8, 4096 * 8, 8192 * 8192 + 8])
def test_gelu_fwd(n):
    g = torch.Generator(device="cuda").manual_seed(n % 1000)
    u = (2 * torch.randn(n, device="cuda", generator=g)).bfloat16()
    y = torch.empty_like(u)
    K.gelu_fwd(u, y)
    close(y, F.gelu(u.float(), approximate="tanh"), atol=1e-3)


def test_ln_bwd_bf16_grads_and_sizes():
    """bf16 dgamma/dbeta/dres_sum outputs; T below one CTA's rows; all H sizes."""
    for T, H in [(3, 128), (5, 256), (17, 8192), (2048, 1024)]:
        g = torch.Generator(device="cuda").manual_seed(T + H)
        x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
        w = torch.ones(H, device="cuda").bfloat16()
        dy = torch.randn(T, H, device="cuda", generator=g).bfloat16()
        dr = torch.randn(T, H, device="cuda", generator=g).bfloat16()
        y, mean, rstd = torch.empty_like(x), torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
        K.ln_fwd(x, w, torch.zeros_like(w), y, mean, rstd)
        dx = torch.empty_like(x)
        dg, db, ds = (torch.empty(H, device="cuda").bfloat16() for _ in range(3))
        K.ln_bwd(dy, x, w, mean, rstd, dx, dg, db, K.Workspace(), dres=dr, dres_sum=ds)
        close(db, dy.float().sum(0), atol=1e-2 * T ** 0.5)
        close(ds, dr.float().sum(0), atol=1e-2 * T ** 0.5)


@pytest.mark.parametrize("T,N", [(8192, 8192), (1000, 2048), (7, 24)])
@pytest.mark.parametrize("gelu", [False, True])
def test_bias_grad(T, N, gelu):
    g = torch.Generator(device="cuda").manual_seed(N)
    dy = torch.randn(T, N, device="cuda", generator=g).bfloat16()
    u = torch.randn(T, N, device="cuda", generator=g).bfloat16() if gelu else None
    du = torch.empty_like(dy) if gelu else None
    db = torch.empty(N, device="cuda").bfloat16()
    K.bias_grad(dy, db, K.Workspace(), u=u, du=du)
    if gelu:
        ref_du = torch.ops.aten.gelu_backward(dy.float(), u.float(), approximate="tanh")
        close(du, ref_du, atol=1e-2)
        ref = du.float().sum(0)
    else:
        ref = dy.float().sum(0)
    close(db, ref, atol=1e-3 * T ** 0.5)


@pytest.mark.parametrize("T,V", [(8, 512), (1024, 50304), (33, 1000), (300, 50304), (5, 1001)])
def test_softmax_ce(T, V):
    g = torch.Generator(device="cuda").manual_seed(V)
    logits = (3 * torch.randn(T, V, device="cuda", generator=g)).bfloat16()
    tgt = torch.randint(0, V, (T,), device="cuda", generator=g)
    lf = logits.float().requires_grad_(True)
    ref_loss = F.cross_entropy(lf, tgt)
    ref_loss.backward()
    work = logits.clone()
    rows = torch.empty(T, device="cuda")
    loss = torch.empty((), device="cuda")
    K.softmax_ce(work, tgt, rows, loss, 1.0 / T)
    assert abs(loss.item() - ref_loss.item()) < 1e-4 * max(1.0, abs(ref_loss.item()))
    close(work, lf.grad, atol=1e-4 / T)


@pytest.mark.parametrize("T,H,dres", [(8192, 2048, True), (300, 4096, True), (513, 1024, False),
                                      (17, 8192, True), (3, 128, False)])
def test_ln_bwd_partials_and_fold_sets_equal_ln_bwd(T, H, dres):
    """zi_ln_bwd_partials + zi_fold_sets (the deferred folds) == zi_ln_bwd, bit for bit,
    with a colsum fold riding in the same zi_fold_sets launch == zi_colsum_fold."""
    g = torch.Generator(device="cuda").manual_seed(T * 7 + H)
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    w = (1 + 0.1 * torch.randn(H, device="cuda", generator=g)).bfloat16()
    dy = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    dr = torch.randn(T, H, device="cuda", generator=g).bfloat16() if dres else None
    y, mean, rstd = torch.empty_like(x), torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
    K.ln_fwd(x, w, torch.zeros_like(w), y, mean, rstd)
    outs = []
    for deferred in (False, True):
        dx = torch.empty_like(x)
        dg, db, ds = (torch.empty(H, device="cuda").bfloat16() for _ in range(3))
        if deferred:
            part = torch.empty(3 * 2 * 148 * H + 1000, device="cuda")
            P = K.ln_bwd_partials(dy, x, w, mean, rstd, dx, part, dres=dr, dres_sum=dres)
            sets = [(part[i * P * H:], P, H, o) for i, o in enumerate((dg, db, ds)[:3 if dres else 2])]
            K.fold_sets(sets)
        else:
            K.ln_bwd(dy, x, w, mean, rstd, dx, dg, db, K.Workspace(), dres=dr, dres_sum=ds if dres else None)
        outs.append((dx, dg, db, ds if dres else dg))
    for a, b in zip(*outs):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    # column partials of another producer folded in the same launch, fp32 outputs
    cp = torch.randn(37, 611, device="cuda", generator=g)
    o1 = torch.empty(611, device="cuda")
    o2 = torch.empty(611, device="cuda")
    o3 = torch.empty(5, device="cuda")
    K.colsum_fold(cp, 37, 611, o1)
    K.fold_sets([(cp, 37, 611, o2), (cp, 2, 5, o3)])
    assert torch.equal(o1, o2)
    assert torch.equal(o3, cp.view(-1)[:5] + cp.view(-1)[5:10])   # part[p * N + c], N = 5
