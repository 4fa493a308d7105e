"""zi_embed_grad: the tied-embedding gradient summed per vocabulary row in sequence order.

Checked against a float64 reference of acc + scatter-add (within one half ulp of the
rounded result) and for bitwise repeatability, including more tokens than one shared
tile (T > 8192) and repeated ids."""

import pytest
import torch

from paper_2104_07857_b200 import kernels

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,V,hd,dt", [(512, 64, 64, torch.bfloat16), (8192, 50304, 256, torch.bfloat16),
                                       (20000, 300, 128, torch.float32)])
def test_embed_grad_matches_scatter_add(T, V, hd, dt):
    g = torch.Generator(device="cuda").manual_seed(T)
    tok = torch.randint(0, V, (T,), device="cuda", generator=g)
    dx = torch.randn(T, hd, device="cuda", generator=g).to(dt)
    acc = torch.randn(V, hd, device="cuda", generator=g)
    work = torch.empty(2 * V + 1 + T, dtype=torch.int32, device="cuda")
    out = torch.empty(V, hd, dtype=torch.bfloat16, device="cuda")
    kernels.embed_grad(tok, dx, acc, out, work)
    ref = acc.double().index_add(0, tok, dx.double())
    # in-order fp32 sum then one bf16 rounding: within a bf16 ulp of the exact value
    assert ((out.double() - ref).abs() <= ref.abs() * 2 ** -7 + 1e-5 * T / V).all()
    out2 = torch.empty_like(out)
    kernels.embed_grad(tok, dx, acc, out2, work)
    assert torch.equal(out.view(torch.int16), out2.view(torch.int16))
    # the sequence-order fold, exactly: row v = fp32(acc[v] + fp32 sum of its dx rows in t order)
    v = int(tok[T // 2])
    rows = (tok == v).nonzero().flatten().tolist()
    s = torch.zeros(hd, dtype=torch.float32, device="cuda")
    for t in rows:
        s = s + dx[t].float()
    assert torch.equal(out[v], (acc[v] + s).bfloat16())


@pytest.mark.parametrize("B,S,V,hd", [(8, 1024, 50304, 2048), (4, 128, 512, 256), (3, 5, 7, 8)])
def test_embed_fwd_equals_torch_lookup_plus_position(B, S, V, hd):
    """zi_embed_fwd == F.embedding(tok, wte) + wpe (torch's bf16 add: fp32 sum, one RNE)."""
    g = torch.Generator(device="cuda").manual_seed(B * S + hd)
    tok = torch.randint(0, V, (B, S), device="cuda", generator=g)
    wte = torch.randn(V, hd, device="cuda", generator=g).bfloat16()
    wpe = torch.randn(S, hd, device="cuda", generator=g).bfloat16()
    x = torch.empty(B * S, hd, dtype=torch.bfloat16, device="cuda")
    kernels.embed_fwd(tok, wte, wpe, x)
    ref = (torch.nn.functional.embedding(tok, wte) + wpe).reshape(-1, hd)
    assert torch.equal(x.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("dxt,outt", [(torch.bfloat16, torch.bfloat16), (torch.bfloat16, torch.float32),
                                      (torch.float32, torch.float16), (torch.float16, torch.bfloat16)])
def test_pos_grad_is_the_in_order_batch_sum(dxt, outt):
    """zi_pos_grad: out[s] = RNE(sum over b ascending of dx[b, s]) with an fp32 sum."""
    B, S, hd = 8, 1024, 2048
    g = torch.Generator(device="cuda").manual_seed(5)
    dx = torch.randn(B * S, hd, device="cuda", generator=g).to(dxt)
    out = torch.empty(S, hd, dtype=outt, device="cuda")
    kernels.pos_grad(dx, B, out)
    s = torch.zeros(S, hd, dtype=torch.float32, device="cuda")
    for b in range(B):
        s = s + dx[b * S:(b + 1) * S].float()
    assert torch.equal(out, s.to(outt))
