"""TierStore drop-in parity with the reference infinisim.store.

CPU: shard files byte-identical to files the REFERENCE wrote (tests/golden/
store_ref, made by tests/golden/make_golden.py), same accounting, and a
differential run of 10^4 random operations against the reference store
itself when /root/reference is present (AC-11). GPU: the full scripted
sequence including the HBM device tier.
"""

import json
import os
import sys

import numpy as np
import pytest
import torch

from paper_2104_07857_b200 import store as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the reference source (build container) or its unmodified install in baseline/_ref
REF_SRC = next((p for p in ("/root/reference/pkg/src", os.path.join(_ROOT, "baseline", "_ref"))
                if os.path.isdir(os.path.join(p, "infinisim"))), "/nonexistent")


def load_gold():
    with open(os.path.join(GOLD, "store_ref.json")) as f:
        return json.load(f)


def gold_arrays(g):
    return {k: np.frombuffer(bytes.fromhex(h), dtype=np.dtype(dt)) for k, (dt, h) in g["arrays"].items()}


def run_script(st, arrays, device_tier: bool):
    T = S.TierKind
    for k, a in arrays.items():
        st.flush([st.write(k, a, T.NVME)])
    if device_tier:
        st.flush([st.write("dev", arrays["a/f32"], T.DEVICE)])
    st.flush([st.write("host", arrays["b/f16"], T.HOST)])
    with pytest.raises(S.CapacityExceeded):
        st.write("big", np.zeros(1000, "<f4"), T.HOST)
    r = st.read_range("a/f32", T.NVME, 5, 10).wait()
    st.flush([st.write_range("b/f16", T.NVME, 3, np.ones(4, "<f2"))])
    if device_tier:
        st.move("dev", T.DEVICE, T.NVME)
    else:
        st.flush([st.write("dev", arrays["a/f32"], T.NVME)])
    return r


@pytest.mark.parametrize("device_tier", [False, pytest.param(True, marks=pytest.mark.gpu)])
def test_script_matches_reference(tmp_path, device_tier):
    g = load_gold()
    arrays = gold_arrays(g)
    pool = S.BufferPool(buffer_bytes=64, buffer_count=2)
    st = S.TierStore(4096, 2048, nvme_root=str(tmp_path), pool=pool, sync_io=True)
    r = run_script(st, arrays, device_tier)
    assert r.numpy().astype("<f4").tobytes().hex() == g["range_a"]
    for fn in os.listdir(os.path.join(GOLD, "store_ref")):
        with open(os.path.join(GOLD, "store_ref", fn), "rb") as f:
            want = f.read()
        with open(os.path.join(tmp_path, fn), "rb") as f:
            assert f.read() == want, fn
    stats = st.stats()
    got = {t.value: [s.capacity, s.used, s.peak_used, s.bytes_read, s.bytes_written]
           for t, s in stats.tiers.items()}
    for tier in (("device", "host", "nvme") if device_tier else ("host", "nvme")):
        if tier == "nvme" and not device_tier:
            continue  # the CPU variant writes "dev" directly instead of moving it
        assert got[tier] == g["stats"][tier], tier
    assert st.keys(S.TierKind.NVME) == g["keys_nvme"]
    assert {k: st.length(k, S.TierKind.NVME) for k in g["keys_nvme"]} == g["lengths"]
    st.close()


@pytest.mark.parametrize("tier", ["host", "nvme"])
def test_read_into_write_from(tmp_path, tier):
    """Engine extensions: range I/O into / from caller tensors, same bytes as read_range."""
    T = S.TierKind(tier)
    st = S.TierStore(0, 1 << 20, nvme_root=str(tmp_path), sync_io=True)
    a = np.arange(1000, dtype=np.float32)
    st.flush([st.write("k", a, T)])
    out = torch.empty(100, dtype=torch.float32)
    st.flush([st.read_into("k", T, out, start=250)])
    assert np.array_equal(out.numpy(), a[250:350])
    st.flush([st.write_from("k", T, 10, torch.full((5,), -1.0))])
    assert np.array_equal(st.read_range("k", T, 8, 9).wait().numpy(),
                          np.array([8, 9, -1, -1, -1, -1, -1, 15, 16], np.float32))
    with pytest.raises(ValueError):
        st.read_into("k", T, torch.empty(10, dtype=torch.float64))
    with pytest.raises(S.KeyNotFound):
        st.read_into("nope", T, out)


def test_buffer_pool_contract():
    p = S.BufferPool(buffer_bytes=16, buffer_count=2, blocking=False, pinned=False)
    a, b = p.acquire(), p.acquire()
    with pytest.raises(S.PoolExhausted):
        p.acquire()
    p.release(a)
    p.release(b)
    with pytest.raises(ValueError):
        p.release(a)  # over-release
    with pytest.raises(ValueError):
        p.release(bytearray(16))  # foreign buffer
    assert p.free_count == 2


def test_buffer_pool_native_blocking_waits():
    """The native pool (zi_pool_*) parks a blocked acquire in C and counts it in waits."""
    import threading
    import time
    p = S.BufferPool(buffer_bytes=32, buffer_count=1, blocking=True, pinned=False)
    a = p.acquire()
    got = []
    t = threading.Thread(target=lambda: got.append(p.acquire()))
    t.start()
    time.sleep(0.2)
    assert not got and p.waits == 1      # parked, GIL released
    p.release(a)
    t.join(5)
    assert got == [a] and p.free_count == 0
    p.release(a)
    assert p.free_count == 1
    # LIFO hand-out like the reference's list.pop()
    q = S.BufferPool(buffer_bytes=8, buffer_count=3, blocking=False, pinned=False)
    x, y = q.acquire(), q.acquire()
    q.release(x)
    assert q.acquire() is x
    v = S._buf_view(y)
    v[:3] = b"abc"
    assert bytes(S._buf_tensor(y)[:3].numpy()) == b"abc"
    q.close()


def test_errors_and_visibility(tmp_path):
    st = S.TierStore(0, 1024, nvme_root=str(tmp_path), sync_io=True)
    with pytest.raises(S.KeyNotFound):
        st.read("missing", S.TierKind.NVME)
    with pytest.raises(KeyError):
        st.read("missing", S.TierKind.HOST)
    with pytest.raises(ValueError):
        st.write("x", np.zeros((2, 2), np.float32), S.TierKind.HOST)
    with pytest.raises(ValueError):
        st.write("x", np.zeros(3, np.int32), S.TierKind.HOST)
    st.flush([st.write("k", np.arange(4, dtype=np.float32), S.TierKind.NVME)])
    path = os.path.join(tmp_path, "k.shard")
    with open(path, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(S.ShardFormatError):
        st.read("k", S.TierKind.NVME).wait()
    # failed move leaves the source intact (destination over capacity)
    st2 = S.TierStore(0, 8, nvme_root=str(tmp_path / "m"), sync_io=True)
    st2.flush([st2.write("s", np.arange(4, dtype=np.float32), S.TierKind.NVME)])
    with pytest.raises(S.CapacityExceeded):
        st2.move("s", S.TierKind.NVME, S.TierKind.HOST)
    assert st2.exists("s", S.TierKind.NVME)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted")
def test_differential_random_ops(tmp_path):
    """AC-11: 10^4 random write/read/range/move/delete ops, ours vs the reference."""
    _differential(tmp_path, ["host", "nvme"], sync_io=True, seed=2024)


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not installed")
@pytest.mark.parametrize("sync_io", [True, False])
def test_differential_random_ops_gpu_path(tmp_path, sync_io):
    """AC-11 on the B200 code path: the DEVICE tier is HBM tensors on the store's CUDA
    stream, HOST is pinned cudaHostAlloc memory with CUDA-event tickets and _settle, NVMe
    goes through the native pinned pool; with sync_io=False the store's worker threads
    and tickets are in play. Same 10^4-op differential against the unmodified reference
    (baseline/_ref), results and per-tier stats equal."""
    assert torch.cuda.is_available()
    _differential(tmp_path, ["device", "host", "nvme"], sync_io=sync_io, seed=2025)


def _host_bytes(v) -> bytes:
    """Bytes of a read result: numpy (reference), or a torch tensor on any device (ours)."""
    if isinstance(v, torch.Tensor):
        v = v.cpu().numpy()
    return np.asarray(v).tobytes()


def _differential(tmp_path, tiers, sync_io: bool, seed: int):
    sys.path.insert(0, REF_SRC)
    import infinisim.store as R
    rng = np.random.default_rng(seed)
    ours = S.TierStore(1 << 16, 1 << 15, nvme_root=str(tmp_path / "o"),
                       pool=S.BufferPool(256, 4), sync_io=sync_io)
    ref = R.TierStore(1 << 16, 1 << 15, nvme_root=str(tmp_path / "r"),
                      pool=R.BufferPool(256, 4), sync_io=sync_io)
    keys = [f"k{i}" for i in range(24)]
    dts = ["<f2", "<f4", "<f8"]

    def outcome(store, mod, op, args):
        T = mod.TierKind
        try:
            if op == "write":
                k, t, a = args
                store.flush([store.write(k, a, T(t))])
                return ("ok",)
            if op == "read":
                k, t = args
                v = store.read(k, T(t)).wait()
                return ("val", _host_bytes(v))
            if op == "range":
                k, t, s, n = args
                v = store.read_range(k, T(t), s, n).wait()
                return ("val", _host_bytes(v))
            if op == "wrange":
                k, t, s, a = args
                store.flush([store.write_range(k, T(t), s, a)])
                return ("ok",)
            if op == "move":
                k, a_, b_ = args
                store.move(k, T(a_), T(b_))
                return ("ok",)
            if op == "delete":
                k, t = args
                store.delete(k, T(t))
                return ("ok",)
        except Exception as e:  # noqa: BLE001
            return ("err", type(e).__name__)

    for i in range(10_000):
        op = rng.choice(["write", "read", "range", "wrange", "move", "delete"], p=[.3, .2, .15, .1, .1, .15])
        k = str(rng.choice(keys))
        t = str(rng.choice(tiers))
        if op == "write":
            a = rng.standard_normal(int(rng.integers(1, 600))).astype(str(rng.choice(dts)))
            args = (k, t, a)
        elif op in ("read", "delete"):
            args = (k, t)
        elif op == "range":
            args = (k, t, int(rng.integers(0, 50)), int(rng.integers(1, 50)))
        elif op == "wrange":
            args = (k, t, int(rng.integers(0, 50)), rng.standard_normal(int(rng.integers(1, 20))).astype(str(rng.choice(dts))))
        else:
            args = (k, t, str(rng.choice(tiers)))
        o1 = outcome(ours, S, op, args)
        o2 = outcome(ref, R, op, args)
        assert o1 == o2, (i, op, args[:2], o1[:2], o2[:2])
        if i % 500 == 0:
            s1, s2 = ours.stats(), ref.stats()
            for t_ in tiers:
                a_, b_ = s1.tiers[S.TierKind(t_)], s2.tiers[R.TierKind(t_)]
                assert (a_.used, a_.peak_used, a_.bytes_read, a_.bytes_written) == \
                       (b_.used, b_.peak_used, b_.bytes_read, b_.bytes_written)
                assert a_.capacity is None or a_.used <= a_.capacity
            assert s1.buffers_free == s1.buffers_total
    for fn in os.listdir(tmp_path / "r"):
        with open(tmp_path / "r" / fn, "rb") as f1, open(tmp_path / "o" / fn, "rb") as f2:
            assert f1.read() == f2.read(), fn
