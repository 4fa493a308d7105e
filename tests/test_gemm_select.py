"""Host logic of the per-site GEMM choice (CPU): operand eligibility and forced modes."""

import torch

from paper_2104_07857_b200 import gemm_select as gs


def test_aligned_operand_contract():
    a = torch.empty(64, 128, dtype=torch.bfloat16)
    assert gs.aligned(a, a.t(), None)                 # K-major and MN-major views
    assert not gs.aligned(a[:, 1:])                   # base off the 16-byte grid
    assert not gs.aligned(torch.empty(64, 130, dtype=torch.bfloat16)[:, :128])  # ld 130
    assert gs.aligned(torch.empty(64, 136, dtype=torch.bfloat16)[:, :128])      # ld 136
    assert not gs.aligned(a[::2, ::2])                # no unit stride


def test_forced_modes_skip_timing(monkeypatch):
    calls = []
    for mode in ("zi", "cublas"):
        monkeypatch.setenv("ZI_GEMM_SELECT", mode)
        assert gs.tune(("site", 1), lambda: calls.append(1), lambda: calls.append(2)) == mode
    assert calls == []                                # nothing ran, nothing cached
    assert ("site", 1) not in gs._CHOICE
