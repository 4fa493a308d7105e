"""``cmd_train``: the SPEC's verified training driver on the B200 harness.

    python -m paper_2104_07857_b200.cli train --model model.cfg --ranks 4 --tier nvme \\
        --steps 50 --seed 7 --nvme-root /tmp/zinf [--baseline-digest base.txt] \\
        [--loss-csv loss.csv] [--digest-out digest.txt]

Writes the ``step,loss`` CSV and prints the final digest (sha256 over the
gathered fp32 master parameters, as oracle/harness.py). Exit codes
(SPEC.md:856): 0 success, 1 usage/config, 3 digest mismatch, 4 storage I/O.

Flat config: ``[section]`` headers, ``key = value``
lines, ``#`` comments, integers with ``_`` separators and K/M/G/T decimal
suffixes. Unknown keys are rejected with an error naming the key.

    [model]
    layers = 3
    layer0.in = 8
    layer0.out = 16
    layer0.act = relu          # identity | relu | gelu-approx
    layer1.tiles = 4           # > 1 makes it a tiled_linear
    tied = 1:2                 # layers sharing one parameter key
    seed = 7
    [run]
    batch = 16
    lr = 0.01
    chunk = 1M                 # chunked_adam_step chunk_elems
"""

from __future__ import annotations

import argparse
import os
import re
import sys

EXIT_OK, EXIT_USAGE, EXIT_MISMATCH, EXIT_IO = 0, 1, 3, 4

_SUFFIX = {"K": 10**3, "M": 10**6, "G": 10**9, "T": 10**12}
_MODEL_KEYS = {"layers", "tied", "seed"}
_LAYER_KEYS = {"in", "out", "act", "tiles"}
_RUN_KEYS = {"batch", "lr", "chunk"}


class ConfigError(ValueError):
    pass


def parse_int(v: str) -> int:
    v = v.strip().replace("_", "")
    if v and v[-1].upper() in _SUFFIX:
        return int(float(v[:-1]) * _SUFFIX[v[-1].upper()])
    return int(v)


def parse_flat(text: str) -> dict:
    """{section: {key: value}} of the flat config format."""
    out: dict = {}
    sec = None
    for n, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        m = re.fullmatch(r"\[(\w+)\]", line)
        if m:
            sec = m.group(1)
            out.setdefault(sec, {})
            continue
        if "=" not in line or sec is None:
            raise ConfigError(f"line {n}: expected 'key = value' inside a [section]")
        k, v = (x.strip() for x in line.split("=", 1))
        out[sec][k] = v
    return out


def model_from_config(cfg: dict):
    from .harness import LayerSpec, ModelSpec
    if "model" not in cfg or not cfg["model"]:
        raise ConfigError("empty [model] section")
    mdl = cfg["model"]
    for k in mdl:
        base = k.split(".", 1)
        if len(base) == 2 and re.fullmatch(r"layer\d+", base[0]):
            if base[1] not in _LAYER_KEYS:
                raise ConfigError(f"unknown key {k!r}")
        elif k not in _MODEL_KEYS:
            raise ConfigError(f"unknown key {k!r}")
    n = parse_int(mdl.get("layers", "0"))
    if n < 1:
        raise ConfigError("layers must be >= 1")
    layers = []
    for i in range(n):
        def g(key, default=None):
            v = mdl.get(f"layer{i}.{key}", default)
            if v is None:
                raise ConfigError(f"missing key 'layer{i}.{key}'")
            return v
        tiles = parse_int(g("tiles", "1"))
        act = g("act", "identity")
        if act not in ("identity", "relu", "gelu-approx"):
            raise ConfigError(f"layer{i}.act: unknown activation {act!r}")
        layers.append(LayerSpec("tiled_linear" if tiles > 1 else "linear", parse_int(g("in")),
                                parse_int(g("out")), act, tiles))
    tied = []
    if "tied" in mdl:
        for pair in mdl["tied"].split(","):
            a, b = pair.split(":")
            tied.append((int(a), int(b)))
    try:
        return ModelSpec(layers, tied, parse_int(mdl.get("seed", "7")))
    except ValueError as e:
        raise ConfigError(str(e)) from None


def cmd_train(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="zinf train", description=__doc__.split("\n\n")[0])
    ap.add_argument("--model", required=True)
    ap.add_argument("--ranks", type=int, default=1)
    ap.add_argument("--tier", choices=["device", "host", "nvme"], default="device")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--baseline-digest")
    ap.add_argument("--nvme-root", default=os.environ.get("INFINISIM_NVME_ROOT"))
    ap.add_argument("--loss-csv")
    ap.add_argument("--digest-out")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK
    try:
        with open(args.model) as f:
            cfg = parse_flat(f.read())
        spec = model_from_config(cfg)
        for k in cfg.get("run", {}):
            if k not in _RUN_KEYS:
                raise ConfigError(f"unknown key {k!r}")
        run = cfg.get("run", {})
        batch = parse_int(run.get("batch", "16"))
        lr = float(run.get("lr", "0.01"))
        chunk = parse_int(run.get("chunk", "1M"))
        if args.ranks < 1 or args.steps < 0:
            raise ConfigError("--ranks must be >= 1 and --steps >= 0")
        if not args.nvme_root:
            raise ConfigError("--nvme-root (or INFINISIM_NVME_ROOT) is required")
    except (OSError, ConfigError, ValueError) as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_USAGE

    import torch

    from . import harness as H
    from .store import StoreError, TierKind, TierStore
    tier = TierKind(args.tier)
    try:
        with TierStore(1 << 40, 1 << 40, nvme_root=args.nvme_root) as store:
            if args.seed is not None:
                spec = H.ModelSpec(spec.layers, spec.tied_pairs, args.seed)
            model = H.init_partitioned(spec, args.ranks, store, H.HarnessPlacement.all(tier))
            x, t = H.synthetic_batch(spec, batch, store.device)
            hyper = H.AdamHyper(lr=lr)
            losses = [H.train_step(model, (x, t), hyper, store, chunk) for _ in range(args.steps)]
            digest = H.digest(model)
    except (StoreError, OSError) as e:
        print(f"storage I/O error: {e}", file=sys.stderr)
        return EXIT_IO
    except ValueError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_USAGE
    if args.loss_csv:
        with open(args.loss_csv, "w", newline="\n") as f:
            f.write("step,loss\n")
            for i, l in enumerate(losses):
                f.write(f"{i},{l!r}\n")
    if args.digest_out:
        with open(args.digest_out, "w") as f:
            f.write(digest + "\n")
    print(digest)
    if args.baseline_digest:
        with open(args.baseline_digest) as f:
            want = f.read().strip()
        if want != digest:
            print(f"digest mismatch: {digest} != baseline {want}", file=sys.stderr)
            return EXIT_MISMATCH
    torch.cuda.synchronize()
    return EXIT_OK


def cmd_plan(argv=None) -> int:
    """Rank the placement strategies for a model on a cluster profile (planner.py)."""
    from . import planner as P
    ap = argparse.ArgumentParser(prog="zinf plan")
    ap.add_argument("--profile", choices=["dgx2", "b200"], default="b200")
    ap.add_argument("--nodes", type=int, default=1)
    ap.add_argument("--nl", type=int, required=True)
    ap.add_argument("--hd", type=int, required=True)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--bsz", type=float, default=1.0)
    ap.add_argument("--ci", type=int, default=1)
    ap.add_argument("--tiling", type=int, default=1)
    try:
        a = ap.parse_args(argv)
        shape = P.ModelShape(a.nl, a.hd, a.heads, a.seq, a.bsz, a.ci)
        cluster = (P.b200 if a.profile == "b200" else P.dgx2)(a.nodes)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK
    except ValueError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_USAGE
    print(f"model {shape.params:.4g} params on {cluster.name} x {cluster.nodes} node(s), "
          f"{cluster.world_size} devices")
    print("strategy,fits,binding,device_GB,host_GB_per_node,nvme_GB_per_node,pred_eff")
    for r in P.recommend(shape, cluster, a.tiling):
        d = r.demand
        print(f"{r.strategy.value},{int(r.fits)},{r.binding_constraint},{d['device'] / 1e9:.2f},"
              f"{d['host'] / 1e9:.2f},{d['nvme'] / 1e9:.2f},{r.predicted_efficiency:.4f}")
    return EXIT_OK


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if argv and argv[0] == "plan":
        return cmd_plan(argv[1:])
    if not argv or argv[0] != "train":
        print("usage: python -m paper_2104_07857_b200.cli {train --model CFG | plan --nl N --hd H}"
              " [options]\n(sweep / simulate are analytic SPEC modules outside this build's hot"
              " path)", file=sys.stderr)
        return EXIT_USAGE
    return cmd_train(argv[1:])


if __name__ == "__main__":
    sys.exit(main())
