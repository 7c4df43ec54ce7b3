"""Random jagged packs through the C-ABI against the numpy restatement of the
reference (prefix = cumsum(lens) cast to the index dtype, collection.py:553-554;
members = the concatenated segments, collection.py:555-556, split per leaf as
import_external does, transfer.py:301-320).

Each case draws a record count, a length distribution (uniform, mostly empty,
one giant record, a block of long records), length and index dtypes, a member
layout (one 4/8-byte field, or 2-4 fields of an 8/16-byte record, or an odd
generic layout), pointer offsets off 16-byte alignment, and a pool capacity
that is sometimes too small. It covers the fused kernel (one field, record
staging, the queue for skewed sub-tiles, overflow) and the two-kernel path
for the layouts the fused kernel does not take."""

import numpy as np
import pytest

from test_gpu_jagged_paths import _expect, _pack

pytestmark = pytest.mark.gpu

LENS_TYPES = [np.int32, np.int64, np.uint32, np.uint16, np.uint8]
PREFIX_TYPES = ["i32", "i64", "u32", "u16"]
LAYOUTS = [
    (8, [(0, 8)]),
    (4, [(0, 4)]),
    (8, [(0, 4), (4, 4)]),
    (16, [(0, 8), (8, 4), (12, 4)]),
    (16, [(4, 4), (8, 8)]),
    (12, [(0, 4), (4, 8)]),       # 8-byte field at an unaligned record offset: two-kernel path
    (6, [(0, 2), (2, 4)]),        # 2-byte field: two-kernel path
]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([0, 1, 7, 1023, 1024, 1025, 40_000, 250_001]))
    ltype = LENS_TYPES[rng.integers(len(LENS_TYPES))]
    cap = int(np.iinfo(ltype).max)
    kind = rng.integers(4)
    if kind == 0:
        lens = rng.integers(0, min(25, cap) + 1, n)
    elif kind == 1:
        lens = (rng.random(n) < 0.05) * rng.integers(1, min(6, cap) + 1, n)
    elif kind == 2:
        lens = rng.integers(0, 4, n)
        if n:
            lens[rng.integers(n)] = min(cap, 90_000)
    else:
        lens = rng.integers(0, 3, n)
        if n > 2000:
            lens[500:1600] = min(cap, 120)   # sub-tiles far over 64 members/record: the shared queue
    lens = lens.astype(ltype)
    stride, fields = LAYOUTS[rng.integers(len(LAYOUTS))]
    ptype = PREFIX_TYPES[rng.integers(len(PREFIX_TYPES))]
    order = rng.permutation(n)
    gaps = lens[order].astype(np.int64) + rng.integers(0, 3, n)
    offs = np.empty(n, np.int64)
    if n:
        offs[order] = np.concatenate([[0], np.cumsum(gaps)[:-1]])
    plen = int(gaps.sum()) if n else 0
    pool = rng.integers(0, 256, max(plen, 1) * stride, dtype=np.uint8)
    T = int(lens.astype(np.int64).sum())
    cap_extra = int(rng.choice([0, 5, -(T // 3) if T > 3 else 0]))
    return dict(lens=lens, offs=offs, pool=pool, stride=stride, fields=fields, ptype=ptype, cap_extra=cap_extra,
                lens_shift=int(rng.integers(2)), prefix_shift=int(rng.integers(2)))


@pytest.mark.parametrize("seed", range(24))
def test_random_packs_match_the_restatement(seed):
    c = _case(seed)
    p, got, t = _pack(c["lens"], c["offs"], c["pool"], c["stride"], c["fields"], c["ptype"], cap_extra=c["cap_extra"],
                      lens_shift=c["lens_shift"], prefix_shift=c["prefix_shift"])
    pw, want, tw = _expect(c["lens"], c["offs"], c["pool"][:max(len(c["pool"]), 0)], c["stride"], c["fields"],
                           c["ptype"])
    assert t == tw
    assert p.tobytes() == pw.tobytes()
    if c["cap_extra"] >= 0:  # within capacity: the pools are complete (past it the caller re-packs)
        assert got == want
