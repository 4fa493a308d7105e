"""cmd_train: flat config parsing (CPU) and the verified run (GPU)."""

import os

import pytest

from paper_2104_07857_b200 import cli

CFG = """
# SPEC AC-9 toy model 8 -> 16 -> 16 -> 4
[model]
layers = 3
layer0.in = 8
layer0.out = 16
layer0.act = relu
layer1.in = 16
layer1.out = 16
layer1.act = relu
layer1.tiles = 4
layer2.in = 16
layer2.out = 4
seed = 7
[run]
batch = 16
lr = 0.01
chunk = 1_000
"""


def test_parse_flat_and_model():
    cfg = cli.parse_flat(CFG)
    spec = cli.model_from_config(cfg)
    assert [l.kind for l in spec.layers] == ["linear", "tiled_linear", "linear"]
    assert spec.layers[1].tiles == 4 and spec.seed == 7
    assert cli.parse_int("1_000") == 1000 and cli.parse_int("2K") == 2000 and cli.parse_int("1M") == 10**6


def test_config_errors(tmp_path):
    with pytest.raises(cli.ConfigError):
        cli.model_from_config(cli.parse_flat("[model]\n"))
    with pytest.raises(cli.ConfigError, match="bogus"):
        cli.model_from_config(cli.parse_flat("[model]\nlayers = 1\nlayer0.in = 2\nlayer0.out = 2\nbogus = 1\n"))
    p = tmp_path / "bad.cfg"
    p.write_text("[model]\n")
    assert cli.main(["train", "--model", str(p), "--nvme-root", str(tmp_path)]) == cli.EXIT_USAGE
    assert cli.main(["plan"]) == cli.EXIT_USAGE


@pytest.mark.gpu
def test_train_digest_verification(tmp_path):
    cfgp = tmp_path / "m.cfg"
    cfgp.write_text(CFG)
    d1 = tmp_path / "d1.txt"
    rc = cli.main(["train", "--model", str(cfgp), "--ranks", "1", "--tier", "device", "--steps", "20",
                   "--nvme-root", str(tmp_path / "a"), "--digest-out", str(d1),
                   "--loss-csv", str(tmp_path / "loss.csv")])
    assert rc == cli.EXIT_OK
    lines = (tmp_path / "loss.csv").read_text().splitlines()
    assert lines[0] == "step,loss" and len(lines) == 21
    # world 4 on the NVMe tier must reproduce the digest (placement invariance)
    rc = cli.main(["train", "--model", str(cfgp), "--ranks", "4", "--tier", "nvme", "--steps", "20",
                   "--nvme-root", str(tmp_path / "b"), "--baseline-digest", str(d1)])
    assert rc == cli.EXIT_OK
    bad = tmp_path / "bad.txt"
    bad.write_text("0" * 64 + "\n")
    rc = cli.main(["train", "--model", str(cfgp), "--steps", "1", "--nvme-root", str(tmp_path / "c"),
                   "--baseline-digest", str(bad)])
    assert rc == cli.EXIT_MISMATCH


@pytest.mark.gpu
def test_corrupt_shard_is_storage_error(tmp_path, monkeypatch):
    """A corrupted NVMe shard surfaces as exit code 4."""
    from paper_2104_07857_b200 import harness as H
    cfgp = tmp_path / "m.cfg"
    cfgp.write_text(CFG)
    root = tmp_path / "n"
    orig = H.train_step

    def corrupting(model, *a, **k):
        for fn in os.listdir(root):
            if fn.endswith(".shard"):
                with open(root / fn, "r+b") as f:
                    f.write(b"JUNK")
        return orig(model, *a, **k)

    monkeypatch.setattr(H, "train_step", corrupting)
    rc = cli.main(["train", "--model", str(cfgp), "--ranks", "2", "--tier", "nvme", "--steps", "1",
                   "--nvme-root", str(root)])
    assert rc == cli.EXIT_IO
