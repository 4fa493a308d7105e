"""Hand-written tcgen05 causal attention (csrc/attn_sm100.cu) against an fp32 torch
reference of the same op, and its backward's determinism.

Forward and backward take bf16 operands and round the probability / gradient tiles
to bf16 before the second MMA (as every flash kernel does), so the comparison with
the fp32 reference is within bf16 resolution: measured worst-case errors are noted
beside each bound. The backward must be bitwise identical across repeated runs
(no atomics, fixed-order sums).
"""

import math

import pytest
import torch

from paper_2104_07857_b200 import kernels

pytestmark = pytest.mark.gpu


def reference(qkv, B, H, S, D):
    q, k, v = qkv.float().view(B, S, 3, H, D).unbind(2)
    q, k, v = (t.transpose(1, 2).requires_grad_(True) for t in (q, k, v))
    s = (q @ k.transpose(-1, -2)) / math.sqrt(D)
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=qkv.device), 1)
    p = torch.softmax(s.masked_fill(mask, float("-inf")), -1)
    o = p @ v
    return o, (q, k, v), torch.logsumexp(s.masked_fill(mask, float("-inf")), -1)


@pytest.mark.parametrize("B,H,S,D", [(1, 1, 128, 64), (2, 3, 256, 64), (2, 2, 384, 128), (2, 2, 512, 128),
                                     (1, 16, 1024, 128), (4, 4, 128, 128)])
def test_attention_matches_fp32_reference(B, H, S, D):
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + S + D)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda", generator=g).bfloat16()
    out = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda", dtype=torch.float32)
    kernels.attn_fwd(qkv, out, lse, B, H)
    o_ref, (q, k, v), lse_ref = reference(qkv, B, H, S, D)
    o_ref_flat = o_ref.detach().transpose(1, 2).reshape(B * S, H * D)
    err = (out.float() - o_ref_flat).abs().max().item()
    assert err < 2e-2, err
    lse2 = lse_ref.detach().reshape(-1) / math.log(2) * 1.0
    assert (lse - lse2).abs().max().item() < 1e-3
    dout = torch.randn(B * S, H * D, device="cuda", generator=g).bfloat16()
    delta = torch.empty_like(lse)
    dqkv = torch.empty_like(qkv)
    kernels.attn_bwd(qkv, out, dout, lse, delta, dqkv, B, H)
    o_ref.backward(dout.float().view(B, S, H, D).transpose(1, 2))
    want = torch.stack([t.grad.transpose(1, 2) for t in (q, k, v)], 2).reshape(B * S, 3 * H * D)
    rel = (dqkv.float() - want).norm() / want.norm()
    assert rel < 2e-2, rel.item()
    per = [(dqkv.float()[:, i * H * D:(i + 1) * H * D] - want[:, i * H * D:(i + 1) * H * D]).abs().max().item()
           for i in range(3)]
    scale = want.abs().max().item()
    assert max(per) < 5e-2 * scale, (per, scale)
    # deterministic: a second backward is bitwise identical
    dqkv2 = torch.empty_like(qkv)
    kernels.attn_bwd(qkv, out, dout, lse, delta, dqkv2, B, H)
    assert torch.equal(dqkv.view(torch.int16), dqkv2.view(torch.int16))
    out2 = torch.empty_like(out)
    kernels.attn_fwd(qkv, out2, lse, B, H)
    assert torch.equal(out.view(torch.int16), out2.view(torch.int16))
    # out = None: delta is taken as given (rowsum(dout o out), here the kernel's own
    # from the first call) and the backward is the same bit for bit
    dqkv3 = torch.empty_like(qkv)
    kernels.attn_bwd(qkv, None, dout, lse, delta, dqkv3, B, H)
    assert torch.equal(dqkv.view(torch.int16), dqkv3.view(torch.int16))
    ref_delta = (out.float() * dout.float()).view(B, S, H, D).sum(-1).permute(0, 2, 1).reshape(-1)
    torch.testing.assert_close(delta, ref_delta, rtol=1e-5, atol=1e-4)
    # with the bias-gradient side output: dqkv unchanged bit for bit, and the 32-row block
    # column sums fold to the column sums of dqkv as stored
    part = torch.full(((B * S) // 32 * 3 * H * D,), float("nan"), device="cuda")
    dqkv4 = torch.empty_like(qkv)
    kernels.attn_bwd(qkv, out, dout, lse, delta, dqkv4, B, H, colsum=part)
    assert torch.equal(dqkv.view(torch.int16), dqkv4.view(torch.int16))
    db = torch.empty(3 * H * D, device="cuda")
    kernels.colsum_fold(part, (B * S) // 32, 3 * H * D, db)
    torch.cuda.synchronize()
    torch.testing.assert_close(db.double(), dqkv.double().sum(0), rtol=1e-5, atol=1e-4 * S ** 0.5)
