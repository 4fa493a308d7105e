"""SPEC train-harness on the GPU: AC-9 placement / world invariance, AC-10, register_external_param,
and agreement with the CPU oracle (oracle/harness.py) within fp32 tolerance."""

import numpy as np
import pytest
import torch

from oracle import harness as oh
from paper_2104_07857_b200 import harness as H
from paper_2104_07857_b200.store import TierKind, TierStore

pytestmark = pytest.mark.gpu


def spec(tied=False):
    L = H.LayerSpec
    if not tied:
        return H.ModelSpec([L("linear", 8, 16, "relu"), L("linear", 16, 16, "relu"),
                            L("linear", 16, 4)], seed=7)
    return H.ModelSpec([L("linear", 8, 16, "relu"), L("tiled_linear", 16, 16, "gelu-approx", tiles=4),
                        L("linear", 16, 16, "relu"), L("linear", 16, 16, "relu"),
                        L("linear", 16, 4)], tied_pairs=[(2, 3)], seed=7)


def ospec(s):
    return oh.ModelSpec([oh.LayerSpec(l.kind, l.in_dim, l.out_dim, l.act, l.tiles) for l in s.layers],
                        list(s.tied_pairs), s.seed)


@pytest.fixture
def store(tmp_path):
    with TierStore(1 << 30, 1 << 30, nvme_root=str(tmp_path)) as st:
        yield st


@pytest.mark.parametrize("tied", [False, True])
def test_ac9_placement_and_world_invariance(tmp_path, tied):
    torch.backends.cuda.matmul.allow_tf32 = False
    s = spec(tied)
    with TierStore(1 << 30, 1 << 30, nvme_root=str(tmp_path / "a")) as st1:
        d1, l1 = H.run_training(s, 1, H.HarnessPlacement.all(TierKind.DEVICE), 50, 7, st1)
    with TierStore(1 << 30, 1 << 30, nvme_root=str(tmp_path / "b")) as st4:
        d4, l4 = H.run_training(s, 4, H.HarnessPlacement.all(TierKind.NVME), 50, 7, st4,
                                chunk_elems=3)
    assert d1 == d4 and l1 == l4
    assert l1[-1] < 0.5 * l1[0]
    od, ol = oh.run_training(ospec(s), 1, 50)
    # same math, different fp32 summation order (cuBLAS vs numpy): tight early,
    # and the trajectories stay together (training amplifies ulp differences)
    np.testing.assert_allclose(l1[:10], ol[:10], rtol=1e-4)
    np.testing.assert_allclose(l1, ol, rtol=2e-2)


def test_host_placement_matches_device(tmp_path):
    torch.backends.cuda.matmul.allow_tf32 = False
    s = spec()
    with TierStore(1 << 30, 1 << 30, nvme_root=str(tmp_path)) as st:
        d1, _ = H.run_training(s, 2, H.HarnessPlacement.all(TierKind.DEVICE), 5, 7, st)
    with TierStore(1 << 30, 1 << 30, nvme_root=str(tmp_path / "h")) as st:
        d2, _ = H.run_training(s, 2, H.HarnessPlacement(TierKind.HOST, TierKind.HOST), 5, 7, st)
    assert d1 == d2


def test_register_external_param(store):
    s = spec(tied=True)
    m = H.init_partitioned(s, 2, store)
    assert "layer2" in m.fetch_sets[3]
    before = set(m.fetch_sets[3])
    H.register_external_param(m, "layer2", 3)   # idempotent
    assert m.fetch_sets[3] == before
    with pytest.raises(KeyError):
        H.register_external_param(m, "nope", 1)
    m.fetch_sets[3].discard("layer2")          # unregistered cross-layer access
    x, t = H.synthetic_batch(s, 16, store.device)
    with pytest.raises(H.MissingParam):
        H.train_step(m, (x, t), H.AdamHyper(), store)


def test_init_partitioned_layout(store):
    """Shards equal the oracle's init (bit-exact), same keys."""
    s = spec(tied=True)
    m = H.init_partitioned(s, 3, store)
    st = oh.init_partitioned(ospec(s), 3)
    assert sorted(m.parts) == sorted(st.p16)
    for key in st.p16:
        for r in range(3):
            got = store.tensor(f"{key}.p32/rank{r}", TierKind.DEVICE).cpu().numpy()
            assert np.array_equal(got, st.p32[key][r])
            h = store.tensor(f"{key}.p16/rank{r}", TierKind.DEVICE).cpu().view(torch.int16).numpy()
            assert np.array_equal(h.view(np.uint16), st.p16[key][r])
