"""Jagged packer (K4): decoupled look-back scan + member gather vs the
reference's jagged_fill / import_external golden vectors and the oracle."""

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, HOST, PINNED
from oracle import restate as R
from paper_2511_04853_b200 import jagged, layouts as ly
from paper_2511_04853_b200 import memctx as mc
from paper_2511_04853_b200 import schema as sc
from paper_2511_04853_b200 import transfer as tr, workloads as wl
from paper_2511_04853_b200.devarray import DeviceArray
from skhelp import golden

pytestmark = pytest.mark.gpu

ITYPES = {"i32": sc.I32, "u8": sc.U8, "u16": sc.U16, "i64": sc.I64}


def _schema(itype):
    return sc.Schema("J", (sc.declare_per_item("seed", sc.U64), sc.declare_jagged("members", itype, sc.U64)))


def _read(coll, path):
    with mc.execution_scope(mc.CUDA):
        return coll.prefix_sums(path), coll.column(path).read()


@pytest.mark.parametrize("label", list(ITYPES))
@pytest.mark.parametrize("ctx", ["cuda", "host"])
@pytest.mark.parametrize("form", ["arrays", "lists"])  # arrays take _segpack, lists the np.asarray path
def test_jagged_fill_matches_reference(label, ctx, form):
    g = golden("jagged.npz")
    lens = g[f"{label}:lens"]
    pool = g[f"{label}:pool_in"]
    n = lens.size
    info = CUDA if ctx == "cuda" else HOST
    c = sk.Collection(_schema(ITYPES[label]), ly.PER_FIELD, info)
    with mc.execution_scope(mc.CUDA if ctx == "cuda" else mc.HOST):
        c.resize(n)
        cuts = np.concatenate([[0], np.cumsum(lens.astype(np.int64))])
        segs = [pool[cuts[i]:cuts[i + 1]] for i in range(n)]
        c.jagged_fill("members", segs if form == "arrays" else [s.tolist() for s in segs])
    if ctx == "cuda":
        p, m = _read(c, "members")
    else:
        p, m = c.prefix_sums("members"), c.column("members").read()
    assert p.dtype == g[f"{label}:prefix"].dtype
    assert p.tobytes() == g[f"{label}:prefix"].tobytes()
    assert np.asarray(m).tobytes() == g[f"{label}:pool"].tobytes()
    assert c.jagged_size("members") == int(lens.astype(np.int64).sum())


def test_multi_leaf_members_match_import_external():
    g = golden("jagged.npz")
    lens = g["hits:lens"]
    n = lens.size
    pool = np.empty(lens.astype(np.int64).sum(), wl.HIT_DTYPE)
    pool["adc"], pool["t"] = g["hits:adc_in"], g["hits:t_in"]
    offsets = np.concatenate([[0], np.cumsum(lens.astype(np.int64))[:-1]])
    c = sk.Collection(wl.CLUSTER2_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.resize(n)
    total = jagged.pack(c, "hits", lens, offsets, pool.view(np.uint8), member_stride=8,
                        member_offsets={"hits.adc": 0, "hits.t": 4})
    assert total == pool.size
    with mc.execution_scope(mc.CUDA):
        assert c.prefix_sums("hits").tobytes() == g["hits:prefix"].tobytes()
        assert c.column("hits.adc").read().tobytes() == g["hits:adc"].tobytes()
        assert c.column("hits.t").read().tobytes() == g["hits:t"].tobytes()


@pytest.mark.parametrize("n", [0, 1, 4095, 4096, 4097, 1_000_000])
def test_shuffled_pool_gather_vs_oracle(n):
    lens, offsets, pool = wl.cluster_inputs(n, seed=n + 1)
    c = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.resize(n)
    d_lens = DeviceArray.from_numpy(lens)
    d_off = DeviceArray.from_numpy(offsets)
    d_pool = DeviceArray.from_numpy(pool)
    total = jagged.pack(c, "members", d_lens, d_off, d_pool)
    p_want, m_want = R.jagged_pack(lens, offsets, pool, np.int32)
    assert total == m_want.size
    p, m = _read(c, "members")
    assert p.tobytes() == p_want.tobytes()
    assert m.tobytes() == m_want.tobytes()


def test_long_and_empty_segments():
    lens = np.array([0, 0, 100_000, 0, 1, 70_000, 0], np.int64)
    offsets = np.array([0, 5, 10, 3, 200_000, 100_010, 7], np.int64)
    pool = np.arange(300_000, dtype=np.uint64)
    c = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.resize(lens.size)
    jagged.pack(c, "members", lens, offsets, pool)
    p_want, m_want = R.jagged_pack(lens, offsets, pool, np.int32)
    p, m = _read(c, "members")
    assert p.tobytes() == p_want.tobytes() and m.tobytes() == m_want.tobytes()


@pytest.mark.parametrize("itype,idx_dtype", [(sc.I32, np.int32), (sc.U8, np.uint8)])
def test_fused_repack_and_overflow_fallback(itype, idx_dtype):
    """Second and later packs run scan+gather in one call bounded by the pool
    capacity; a pack that outgrows it falls back to scan / grow / gather."""
    schema = sc.Schema("J", (sc.declare_per_item("seed", sc.U64), sc.declare_jagged("members", itype, sc.U64)))
    c = sk.Collection(schema, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.resize(3000)
    for seed, max_len in ((1, 10), (2, 10), (3, 4), (4, 30), (5, 30)):  # 4: overflow, 5: fused again
        lens, offsets, pool = wl.cluster_inputs(3000, seed=seed, max_len=max_len)
        total = jagged.pack(c, "members", lens, offsets, pool)
        p_want, m_want = R.jagged_pack(lens, offsets, pool, idx_dtype)
        p, m = _read(c, "members")
        assert total == m_want.size and c.jagged_size("members") == total
        assert p.tobytes() == p_want.tobytes() and m.tobytes() == m_want.tobytes(), seed


def test_packed_collection_transfers_to_host_aos():
    lens, offsets, pool = wl.cluster_inputs(5000, seed=3)
    c = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.resize(5000)
    jagged.pack(c, "members", lens, offsets, pool)
    h = sk.Collection(wl.CLUSTER_SCHEMA, ly.AOS, PINNED)
    tr.copy_collection(h, c)
    p_want, m_want = R.jagged_pack(lens, offsets, pool, np.int32)
    assert h.prefix_sums("members").tobytes() == p_want.tobytes()
    assert h.column("members").read().tobytes() == m_want.tobytes()
