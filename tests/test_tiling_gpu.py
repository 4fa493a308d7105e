"""Memory-centric tiling on the GPU (AC-8): tiled forward/backward vs the dense oracle."""

import numpy as np
import pytest
import torch

from oracle import tiling as ot
from paper_2104_07857_b200 import tiling as T
from paper_2104_07857_b200.store import TierKind, TierStore

pytestmark = pytest.mark.gpu


@pytest.fixture
def store(tmp_path):
    with TierStore(8 << 30, 1 << 30, nvme_root=str(tmp_path)) as st:
        yield st


@pytest.mark.parametrize("tiles", [1, 2, 3, 4, 7, 16])
@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, 1e-5)])
@pytest.mark.parametrize("world", [1, 3])
def test_tiling_equivalence(store, tiles, dtype, tol, world):
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator().manual_seed(tiles)
    W = torch.randn(128, 512, generator=g, dtype=dtype)
    b = torch.randn(128, generator=g, dtype=dtype)
    x = torch.randn(16, 512, generator=g, dtype=dtype)
    gy = torch.randn(16, 128, generator=g, dtype=dtype)
    tl = T.tile_linear(W.cuda(), b.cuda(), tiles, store, TierKind.DEVICE, key=f"L{tiles}{world}{dtype}",
                       world_size=world)
    assert [e - s for s, e in tl.rows] == [e - s for s, e in ot.tile_rows(128, tiles)]
    y = T.forward_tiled(tl, x.cuda(), store).cpu().numpy()
    yd = ot.forward_tiled(W.numpy(), b.numpy(), x.numpy(), tiles)
    assert np.abs(y - yd).max() / np.abs(yd).max() < tol
    dW, db, dx = T.backward_tiled(tl, x.cuda(), gy.cuda(), store)
    oW, ob, ox = ot.backward_tiled(W.numpy(), x.numpy(), gy.numpy(), tiles)
    gw = np.concatenate([d.cpu().numpy() for d in dW if d is not None])
    assert np.abs(gw - oW).max() / np.abs(oW).max() < tol
    assert np.abs(dx.cpu().numpy() - ox).max() / np.abs(ox).max() < tol


def test_tiles_roundtrip_and_peak(store):
    W = torch.randn(10, 8, device="cuda")
    b = torch.randn(10, device="cuda")
    tl = T.tile_linear(W, b, 4, store, TierKind.HOST, key="rt")
    assert [e - s for s, e in tl.rows] == [3, 3, 3, 1]
    x = torch.zeros(5, 8, device="cuda")
    y = T.forward_tiled(tl, x, store, prefetch=False)
    assert torch.equal(y, b.expand(5, 10))                      # x = 0 -> bias replicated
    f = T.forward_tiled.last_fetcher
    assert f.peak_resident <= -(-(10 * 9 * 4) // 4) + 4 * 9     # ceil(untiled/T) + one row


@pytest.mark.parametrize("tiles", [4, 8, 16])
def test_bf16_tiled_linear_tcgen05(store, tiles):
    """The config-4 operator (scaled down): bf16 tiles on zi_linear_fwd."""
    M, K, Nout = 512, 1024, 4096
    W = (torch.randn(Nout, K, device="cuda") * K ** -0.5).bfloat16()
    b = torch.randn(Nout, device="cuda").bfloat16()
    x = torch.randn(M, K, device="cuda").bfloat16()
    tl = T.tile_linear(W, b, tiles, store, TierKind.DEVICE, key=f"bf{tiles}", world_size=2)
    y = T.forward_tiled(tl, x, store)
    ref = x.float() @ W.float().t() + b.float()
    err = (y.float() - ref).abs()
    assert (err <= ref.abs() * 2 ** -7 + 2e-2).all()
    gy = torch.randn(M, Nout, device="cuda").bfloat16()
    dW, db, dx = T.backward_tiled(tl, x, gy, store)
    rW = gy.float().t() @ x.float()
    rx = gy.float() @ W.float()
    gw = torch.cat([d for d in dW if d is not None]).float()
    assert ((gw - rW).abs() <= rW.abs() * 2 ** -7 + M * 2 ** -20).all()
    assert ((dx.float() - rx).abs() <= rx.abs() * 2 ** -7 + Nout * 2 ** -20).all()
