"""Host packing for Collection.jagged_fill (csrc/segpack.cpp): lengths, starts and
pool equal to the np.asarray + concatenate + cumsum path of the reference
(collection.py:537-556)."""

import numpy as np
import pytest

from paper_2511_04853_b200 import _segpack


def _split(out, n, dt):
    b = np.frombuffer(out, np.uint8)
    return b[:8 * n].view(np.int64), b[8 * n:16 * n].view(np.int64), b[16 * n:].view(dt)


@pytest.mark.parametrize("dt", [np.uint8, np.int32, np.uint64, np.float64])
@pytest.mark.parametrize("n", [500, 200_000])  # one thread / several
def test_pack_matches_concatenate(dt, n):
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 9, n)
    base = rng.integers(0, 100, int(lens.sum())).astype(dt)
    cuts = np.concatenate([[0], np.cumsum(lens)])
    segs = [base[cuts[i]:cuts[i + 1]] for i in rng.permutation(n)]
    out = _segpack.pack_segments(segs, np.dtype(dt))
    L, S, P = _split(out, n, dt)
    assert L.tolist() == [s.size for s in segs]
    assert S.tolist() == np.concatenate([[0], np.cumsum(L)[:-1]]).tolist()
    assert P.tobytes() == np.concatenate(segs).tobytes()


def test_views_empty_and_alloc():
    base = np.arange(100, dtype=np.uint64)
    segs = [base[3:9], base[0:0], base[50:51], base[10:40]]
    asked = []

    def alloc(nbytes):
        asked.append(nbytes)
        return np.full(nbytes + 5, 0xAB, np.uint8)  # larger than asked is fine

    out = _segpack.pack_segments(segs, np.uint64, alloc)
    assert asked == [4 * 16 + 37 * 8]
    L, S, P = _split(np.asarray(out)[:asked[0]], 4, np.uint64)
    assert L.tolist() == [6, 0, 1, 30] and S.tolist() == [0, 6, 6, 7]
    assert P.tolist() == base[3:9].tolist() + [50] + base[10:40].tolist()
    assert _segpack.pack_segments([], np.uint64) == bytearray()


@pytest.mark.parametrize("segs", [
    [np.arange(3, dtype=np.int32)],                    # other dtype: np.asarray converts it
    [[1, 2, 3]],                                       # a list
    [np.arange(6, dtype=np.uint64)[::2]],              # not contiguous
    [np.arange(3, dtype=">u8")],                       # byte-swapped
    [np.zeros((2, 2), np.uint64)],                     # 2-D
    [np.arange(3, dtype=np.uint64)] * 100_000 + [[1]],  # the odd one out, in the last thread's chunk
])
def test_declines_what_needs_conversion(segs):
    assert _segpack.pack_segments(segs, np.uint64) is None


def test_errors():
    with pytest.raises(TypeError):
        _segpack.pack_segments(5, np.uint64)
    with pytest.raises(ValueError):
        _segpack.pack_segments([np.arange(4, dtype=np.uint64)], np.uint64, lambda nb: bytearray(nb - 1))
    with pytest.raises(BufferError):
        _segpack.pack_segments([np.arange(4, dtype=np.uint64)], np.uint64, lambda nb: b"x" * nb)  # read-only


def test_split_views_match_slices():
    pool = np.arange(1000, dtype=np.uint64)
    b = np.array([0, 3, 3, 10, 999, 1000], np.int64)
    v = _segpack.split_views(pool, b)
    assert [x.tolist() for x in v] == [pool[b[i]:b[i + 1]].tolist() for i in range(5)]
    assert all(x.base is not None for x in v) and v[1].size == 0
    assert _segpack.split_views(pool, np.zeros(1, np.int64)) == []
    with pytest.raises(ValueError):
        _segpack.split_views(pool, np.array([0, 5, 3], np.int64))  # out of order
    with pytest.raises(ValueError):
        _segpack.split_views(pool, np.array([0, 1001], np.int64))  # past the pool
