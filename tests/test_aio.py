"""Native file I/O engine (zi_aio_*) on CPU: ragged byte ranges of a reference-format shard
file read and written through O_DIRECT whole blocks + buffered edges."""

import os

import numpy as np
import pytest

from paper_2104_07857_b200 import store as S
from paper_2104_07857_b200.aio import AioEngine, data_offset


def _engine_or_skip(path):
    eng = AioEngine(4)
    try:
        fds = eng.open(path, write=True)
    except OSError as e:   # a filesystem without O_DIRECT (tmpfs / overlay)
        eng.close()
        pytest.skip(f"O_DIRECT unavailable here: {e}")
    return eng, fds


def test_ranges_round_trip(tmp_path):
    n = 3 * 1024 * 1024 + 77                      # ragged: payload not block-multiple
    a = np.random.default_rng(0).standard_normal(n).astype(np.float32)
    with S.TierStore(0, 0, nvme_root=str(tmp_path), sync_io=True) as st:
        st.flush([st.write("w", a, S.TierKind.NVME)])
        path = st._nvme_path("w")
    eng, fds = _engine_or_skip(path)
    pool = S.BufferPool(8 << 20, 2, pinned=False)
    buf, buf2 = pool.acquire(), pool.acquire()
    rng = np.random.default_rng(1)
    try:
        for s, m in [(0, 1), (0, 1019), (1019, 1024), (5, 100_000), (n - 3, 3),
                     (int(rng.integers(0, n - 1_000_000)), 1_000_000)]:
            b0 = S.SHARD_HEADER_BYTES + 4 * s
            eng.wait(eng.submit(fds, False, buf.ptr, b0, b0 + 4 * m))
            d = data_offset(b0)
            got = np.frombuffer(bytes(S._buf_view(buf)[d:d + 4 * m]), np.float32)
            assert np.array_equal(got, a[s:s + m]), (s, m)
        # overwrite two adjacent ragged ranges concurrently (they share an edge block)
        s1, m1, m2 = 4093, 70_001, 50_003
        new = rng.standard_normal(m1 + m2).astype(np.float32)
        ids = []
        for s, part, bb in ((s1, new[:m1], buf), (s1 + m1, new[m1:], buf2)):
            b0 = S.SHARD_HEADER_BYTES + 4 * s
            d = data_offset(b0)
            S._buf_view(bb)[d:d + part.nbytes] = part.tobytes()
            ids.append(eng.submit(fds, True, bb.ptr, b0, b0 + part.nbytes))
        for i in ids:
            eng.wait(i)
        a[s1:s1 + m1 + m2] = new
    finally:
        AioEngine.close_file(fds)
        eng.close()
        pool.release(buf)
        pool.release(buf2)
    raw = open(path, "rb").read()
    assert raw[:4] == S.SHARD_MAGIC and len(raw) == S.SHARD_HEADER_BYTES + 4 * n
    assert np.array_equal(np.frombuffer(raw[S.SHARD_HEADER_BYTES:], np.float32), a)


def test_short_read_is_oserror(tmp_path):
    p = str(tmp_path / "small.bin")
    with open(p, "wb") as f:
        f.write(os.urandom(10_000))
    eng, fds = _engine_or_skip(p)
    pool = S.BufferPool(1 << 20, 1, pinned=False)
    buf = pool.acquire()
    try:
        with pytest.raises(OSError):
            eng.wait(eng.submit(fds, False, buf.ptr, 0, 20_000))
    finally:
        AioEngine.close_file(fds)
        eng.close()
        pool.release(buf)
