"""Regenerate the golden fixtures in tests/golden/ (run in the build container).

* ``store_ref/`` — shard files written by the REFERENCE ``infinisim.store``
  (imported from /root/reference/pkg/src; that path exists only in the
  build container, never on the GPU box) plus ``store_ref.json`` with the
  reference's observable accounting for a scripted sequence of operations.
* ``spec_examples.json`` — the SPEC's own known-answer examples for the
  hot-path functions and the oracle values they
  produce.

Usage: python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def store_script(store_mod, root):
    """Scripted operations on a reference TierStore; returns its observations."""
    S = store_mod
    obs = {}
    pool = S.BufferPool(buffer_bytes=64, buffer_count=2)
    st = S.TierStore(device_capacity=4096, host_capacity=2048, nvme_root=root, pool=pool,
                     sync_io=True)
    rng = np.random.default_rng(11)
    arrays = {
        "a/f32": rng.standard_normal(37).astype("<f4"),
        "b/f16": rng.standard_normal(100).astype("<f2"),
        "c f64%": rng.standard_normal(9).astype("<f8"),
    }
    for k, a in arrays.items():
        st.flush([st.write(k, a, S.TierKind.NVME)])
    st.flush([st.write("dev", arrays["a/f32"], S.TierKind.DEVICE)])
    st.flush([st.write("host", arrays["b/f16"], S.TierKind.HOST)])
    try:
        st.write("big", np.zeros(1000, "<f4"), S.TierKind.HOST)
        obs["host_capacity_error"] = None
    except S.CapacityExceeded as e:
        obs["host_capacity_error"] = type(e).__name__
    r = st.read_range("a/f32", S.TierKind.NVME, 5, 10).wait()
    obs["range_a"] = r.astype("<f4").tobytes().hex()
    st.flush([st.write_range("b/f16", S.TierKind.NVME, 3, np.ones(4, "<f2"))])
    st.move("dev", S.TierKind.DEVICE, S.TierKind.NVME)
    stats = st.stats()
    obs["stats"] = {t.value: [s.capacity, s.used, s.peak_used, s.bytes_read, s.bytes_written]
                    for t, s in stats.tiers.items()}
    obs["keys_nvme"] = st.keys(S.TierKind.NVME)
    obs["lengths"] = {k: st.length(k, S.TierKind.NVME) for k in obs["keys_nvme"]}
    st.close()
    return arrays, obs


def main():
    sys.path.insert(0, ROOT)
    from oracle import numerics as nx
    from oracle.adam import AdamConsts, adam_update
    from oracle.partition import partition, shard_len
    from oracle.tiling import tile_rows

    # ---- reference store fixtures
    sys.path.insert(0, REF_SRC)
    import infinisim.store as ref_store  # noqa: E402  (reference, build container only)
    out_dir = os.path.join(HERE, "store_ref")
    shutil.rmtree(out_dir, ignore_errors=True)
    os.makedirs(out_dir)
    tmp = tempfile.mkdtemp()
    arrays, obs = store_script(ref_store, tmp)
    for fn in sorted(os.listdir(tmp)):
        shutil.copy(os.path.join(tmp, fn), os.path.join(out_dir, fn))
    obs["arrays"] = {k: [str(a.dtype), a.tobytes().hex()] for k, a in arrays.items()}
    with open(os.path.join(HERE, "store_ref.json"), "w") as f:
        json.dump(obs, f, indent=1, sort_keys=True)

    # ---- SPEC examples
    ex = {}
    ex["shard_len"] = [[10, 4, shard_len(10, 4)], [10, 1, shard_len(10, 1)], [1, 17, shard_len(1, 17)]]
    ex["partition_10_4_last_pad"] = int((partition(np.arange(1, 11, dtype=np.float32), 4)[3] == 0).sum())
    ex["tile_rows_10_4"] = [e - s for s, e in tile_rows(10, 4)]
    c = AdamConsts.make(0.1, 0.9, 0.999, 1e-8, 1)
    P, M, V = adam_update(np.ones(1, np.float32), np.zeros(1, np.float32), np.zeros(1, np.float32),
                          np.ones(1, np.float32), c)
    ex["adam_hand"] = {"p": float(P[0]), "m": float(M[0]), "v": float(V[0]),
                       "p_bits": int(P.view(np.uint32)[0])}
    ex["uniform_init_seed7_stream65_first16"] = nx.uniform_init(7, 65, 0, 16, 1 / 2048 ** 0.5).view(
        np.uint32).tolist()
    ex["bf16_rne"] = {str(x): int(nx.f32_to_bf16_bits(np.array([x], np.float32))[0])
                      for x in (1.0, 1.00390625, 1.01171875, -2.5, 3.4e38)}
    with open(os.path.join(HERE, "spec_examples.json"), "w") as f:
        json.dump(ex, f, indent=1, sort_keys=True)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
