"""K4 kernel paths through the C-ABI: reduce-then-scan and look-back scans,
the async (cp.async + bulk store) gather for 4/8-byte members, the register
gather (misaligned destination), the generic multi-field table, wrapping
narrow prefixes and sk_jagged_scatter over a caller-provided prefix.

Oracle: prefix = cumsum(lens) cast to the index dtype (collection.py:553-554),
members = the concatenated segments (collection.py:555-556), restated with
numpy (np.repeat) so multi-million-record cases check in seconds."""

import ctypes as C

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat
from paper_2511_04853_b200 import jagged, layouts as ly
from paper_2511_04853_b200 import memctx as mc
from paper_2511_04853_b200 import workloads as wl
from paper_2511_04853_b200.devarray import DeviceArray
from paper_2511_04853_b200.errors import BoundsError

pytestmark = pytest.mark.gpu

CUDA = mc.ContextInfo.cuda(0)
TC = nat.TYPE_CODES


def _inputs(n, max_len, seed, slack=3):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len + 1, n).astype(np.int32)
    order = rng.permutation(n)
    gaps = lens[order].astype(np.int64) + rng.integers(0, slack + 1, n)
    offs = np.empty(n, np.int64)
    offs[order] = np.concatenate([[0], np.cumsum(gaps)[:-1]]) if n else gaps
    return lens, offs, int(gaps.sum()) if n else 0


def _gather_index(lens, offs):
    """source member index of every output member"""
    P = np.concatenate([[0], np.cumsum(lens.astype(np.int64))])
    T = int(P[-1])
    return np.repeat(offs - P[:-1], lens.astype(np.int64)) + np.arange(T, dtype=np.int64), P


def _pack(lens, offs, pool_bytes, stride, fields, ptype, cap_extra=0, dst_shift=0, lens_shift=0, prefix_shift=0):
    """run sk_jagged_pack; fields = [(offset, size)]; returns (prefix, [field arrays as bytes], total).
    lens_shift / prefix_shift: pass the lengths / prefix that many elements into their buffers
    (off the 16-byte alignment the vector paths use)"""
    n = lens.size
    T = int(lens.astype(np.int64).sum())
    cap = T + cap_extra
    d_lens = DeviceArray.from_numpy(np.concatenate([np.zeros(lens_shift, lens.dtype), lens]), CUDA)
    d_offs = DeviceArray.from_numpy(offs, CUDA)
    d_pool = DeviceArray.from_numpy(pool_bytes, CUDA)
    pnp = np.dtype({"i32": np.int32, "u16": np.uint16, "u8": np.uint8, "i64": np.int64, "u32": np.uint32}[ptype])
    prefix = DeviceArray(n + 1 + prefix_shift, pnp, CUDA)
    outs = [DeviceArray(max(cap, 1) * sz + 64, np.uint8, CUDA) for _, sz in fields]
    need = C.c_size_t(0)
    nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
    sbytes = -(-need.value // 256) * 256 + ((cap + 255) // 256 + 1) * 8
    scratch = DeviceArray(sbytes, np.uint8, CUDA)
    total = DeviceArray(2, np.int64, CUDA)
    nf = len(fields)
    foff = (C.c_int64 * nf)(*[o for o, _ in fields])
    fsz = (C.c_int32 * nf)(*[sz for _, sz in fields])
    dst = (C.c_void_p * nf)(*[o.ptr + dst_shift for o in outs])
    lcode = {np.dtype(np.int32): "i32", np.dtype(np.uint8): "u8", np.dtype(np.uint16): "u16",
             np.dtype(np.int64): "i64", np.dtype(np.uint32): "u32"}[lens.dtype]
    nat.call("sk_jagged_pack", n, d_lens.ptr + lens_shift * lens.dtype.itemsize, TC[lcode],
             prefix.ptr + prefix_shift * pnp.itemsize, TC[ptype], d_offs.ptr, d_pool.ptr, pool_bytes.size // stride,
             stride, nf,
             foff, fsz, dst, cap, scratch.ptr, scratch.n, total.ptr, nat.stream(0))
    nat.sync(0)
    t, bad = (int(v) for v in total.numpy())
    assert bad == 0
    res = [o.numpy()[dst_shift:dst_shift + t * sz].tobytes() for o, (_, sz) in zip(outs, fields)]
    p = prefix.numpy()[prefix_shift:]
    for a in (d_lens, d_offs, d_pool, prefix, scratch, total, *outs):
        a.free()
    return p, res, t


def _expect(lens, offs, pool_bytes, stride, fields, ptype):
    idx, P = _gather_index(lens, offs)
    rec = pool_bytes.reshape(-1, stride)
    want = [rec[idx, o:o + sz].tobytes() for o, sz in fields]
    return P.astype(np.dtype({"i32": np.int32, "u16": np.uint16, "u8": np.uint8, "i64": np.int64,
                              "u32": np.uint32}[ptype])), want, int(P[-1])


@pytest.mark.parametrize("n,max_len,msize", [(1, 5, 8), (300, 20, 8), (1_000_000, 20, 8), (1_000_000, 20, 4),
                                             (200_000, 0, 8), (50_000, 3000, 8)])
def test_async_gather_single_field(n, max_len, msize):
    lens, offs, plen = _inputs(n, max_len, seed=n + max_len)
    pool = np.random.default_rng(1).integers(0, 256, plen * msize + 8, dtype=np.uint8)
    fields = [(0, msize)]
    p, got, t = _pack(lens, offs, pool, msize, fields, "i32", cap_extra=777)
    pw, want, tw = _expect(lens, offs, pool[:plen * msize], msize, fields, "i32")
    assert t == tw
    assert p.tobytes() == pw.tobytes()
    assert got == want


def test_register_gather_misaligned_destination():
    lens, offs, plen = _inputs(400_000, 20, seed=3)
    pool = np.random.default_rng(2).integers(0, 256, plen * 8, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, 8, [(0, 8)], "i32", dst_shift=8)  # dst % 16 == 8 -> register path
    pw, want, _ = _expect(lens, offs, pool, 8, [(0, 8)], "i32")
    assert p.tobytes() == pw.tobytes() and got == want


def test_generic_field_table_unaligned_stride():
    lens, offs, plen = _inputs(100_000, 12, seed=4)
    stride = 15
    fields = [(0, 4), (4, 8), (12, 2), (14, 1)]
    pool = np.random.default_rng(3).integers(0, 256, plen * stride, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, stride, fields, "i64")
    pw, want, _ = _expect(lens, offs, pool, stride, fields, "i64")
    assert p.tobytes() == pw.tobytes() and got == want


def test_wrapping_u16_prefix_uses_wide_gather():
    lens, offs, plen = _inputs(30_000, 9, seed=5)  # ~135k members: the u16 prefix wraps
    pool = np.random.default_rng(4).integers(0, 256, plen * 8, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, 8, [(0, 8)], "u16")
    pw, want, tw = _expect(lens, offs, pool, 8, [(0, 8)], "u16")
    assert tw > 65535 and t == tw
    assert p.tobytes() == pw.tobytes() and got == want


def test_lookback_scan_beyond_direct_grid():
    # > 4096 scan tiles of 4096 lengths: the single-pass look-back scan
    n = 4096 * 4096 + 12345
    lens = (np.random.default_rng(6).integers(0, 4, n)).astype(np.int32)
    d_lens = DeviceArray.from_numpy(lens, CUDA)
    prefix = DeviceArray(n + 1, np.int64, CUDA)
    need = C.c_size_t(0)
    nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
    scratch = DeviceArray(need.value, np.uint8, CUDA)
    total = DeviceArray(1, np.int64, CUDA)
    nat.call("sk_jagged_scan", n, d_lens.ptr, TC["i32"], prefix.ptr, TC["i64"], scratch.ptr, scratch.n, total.ptr,
             nat.stream(0))
    nat.sync(0)
    want = np.concatenate([[0], np.cumsum(lens.astype(np.int64))])
    assert int(total.numpy()[0]) == int(want[-1])
    assert np.array_equal(prefix.numpy(), want)
    for a in (d_lens, prefix, scratch, total):
        a.free()


def test_scatter_over_given_prefix():
    lens, offs, plen = _inputs(250_000, 20, seed=7)
    pool = np.random.default_rng(8).integers(0, 256, plen * 8, dtype=np.uint8)
    P = np.concatenate([[0], np.cumsum(lens.astype(np.int64))]).astype(np.int32)
    T = int(P[-1])
    d_p, d_o, d_pool = (DeviceArray.from_numpy(x, CUDA) for x in (P, offs, pool))
    out = DeviceArray(T * 8, np.uint8, CUDA)
    foff, fsz, dst = (C.c_int64 * 1)(0), (C.c_int32 * 1)(8), (C.c_void_p * 1)(out.ptr)
    nat.call("sk_jagged_scatter", lens.size, d_p.ptr, TC["i32"], d_o.ptr, d_pool.ptr, 8, 1, foff, fsz, dst, T,
             nat.stream(0))
    nat.sync(0)
    _, want, _ = _expect(lens, offs, pool, 8, [(0, 8)], "i32")
    assert out.numpy().tobytes() == want[0]
    for a in (d_p, d_o, d_pool, out):
        a.free()


# ---- fused single-pass pack (one aligned 4/8-byte field, 16-byte-aligned pool) ----

def _skewed_inputs(n, seed):
    """mostly short segments, one block of long ones (a tile over the queueing
    threshold) and a single giant segment"""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 6, n).astype(np.int32)
    lens[1000:1700] = 2000          # ~1.4M members over two or three tiles: queued and shared out
    lens[n // 2] = 700_000           # one record alone over the threshold
    lens[n - 300:] = 0               # trailing empty records
    order = rng.permutation(n)
    gaps = lens[order].astype(np.int64) + rng.integers(0, 3, n)
    offs = np.empty(n, np.int64)
    offs[order] = np.concatenate([[0], np.cumsum(gaps)[:-1]])
    return lens, offs, int(gaps.sum())


@pytest.mark.parametrize("msize", [8, 4])
def test_fused_pack_skewed_lengths_queue_path(msize):
    lens, offs, plen = _skewed_inputs(200_000, seed=11)
    pool = np.random.default_rng(12).integers(0, 256, plen * msize, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, msize, [(0, msize)], "i64", cap_extra=5)
    pw, want, tw = _expect(lens, offs, pool, msize, [(0, msize)], "i64")
    assert t == tw and p.tobytes() == pw.tobytes() and got == want


def test_fused_pack_all_empty_and_single_record():
    lens = np.zeros(300_000, np.int32)
    offs = np.zeros(300_000, np.int64)
    pool = np.zeros(64, np.uint8)
    p, got, t = _pack(lens, offs, pool, 8, [(0, 8)], "i32")
    assert t == 0 and not p.any()
    lens1 = np.array([123_457], np.int32)
    pool1 = np.random.default_rng(1).integers(0, 256, (123_457 + 9) * 8, dtype=np.uint8)
    offs1 = np.array([9], np.int64)
    p, got, t = _pack(lens1, offs1, pool1, 8, [(0, 8)], "u32")
    _, want, tw = _expect(lens1, offs1, pool1, 8, [(0, 8)], "u32")
    assert t == tw and p.tolist() == [0, 123_457] and got == want


def test_fused_pack_overflow_reports_total():
    lens, offs, plen = _inputs(100_000, 20, seed=13)
    T = int(lens.sum())
    pool = np.random.default_rng(14).integers(0, 256, plen * 8, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, 8, [(0, 8)], "i32", cap_extra=-T // 2)
    assert t == T  # the caller sees total > capacity and re-packs
    pw, _, _ = _expect(lens, offs, pool, 8, [(0, 8)], "i32")
    assert p.tobytes() == pw.tobytes()  # the prefix is complete either way


_SUB = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import test_gpu_jagged_paths as T
for n, ml, ms, pt in [(1, 5, 8, 'i32'), (777, 20, 4, 'u16'), (1_000_000, 20, 8, 'i32'), (300_000, 9, 4, 'u16')]:
    lens, offs, plen = T._inputs(n, ml, seed=n)
    pool = np.random.default_rng(2).integers(0, 256, plen * ms + 8, dtype=np.uint8)
    p, got, t = T._pack(lens, offs, pool, ms, [(0, ms)], pt, cap_extra=3)
    pw, want, tw = T._expect(lens, offs, pool[:plen * ms], ms, [(0, ms)], pt)
    assert t == tw and p.tobytes() == pw.tobytes() and got == want, (n, ml, ms, pt)
lens, offs, plen = T._skewed_inputs(200_000, seed=3)
pool = np.random.default_rng(4).integers(0, 256, plen * 8, dtype=np.uint8)
p, got, t = T._pack(lens, offs, pool, 8, [(0, 8)], 'i64')
pw, want, tw = T._expect(lens, offs, pool, 8, [(0, 8)], 'i64')
assert t == tw and p.tobytes() == pw.tobytes() and got == want
print('ok')
"""


@pytest.mark.parametrize("env", [{"SK_JAGGED_FUSED": "0"}])
def test_pack_variants_in_subprocess(env):
    """the two-kernel path (scan, then gather) on the fused path's cases"""
    import os
    import subprocess
    import sys

    tests = os.path.dirname(os.path.abspath(__file__))
    code = _SUB.format(root=os.path.dirname(tests), tests=tests)
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("ltype", [np.uint8, np.uint16, np.int64, np.uint32])
def test_fused_pack_length_types(ltype):
    lens, offs, plen = _inputs(150_001, 20, seed=21)
    lens = lens.astype(ltype)
    pool = np.random.default_rng(22).integers(0, 256, plen * 8, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, 8, [(0, 8)], "i64", cap_extra=1)
    pw, want, tw = _expect(lens, offs, pool, 8, [(0, 8)], "i64")
    assert t == tw and p.tobytes() == pw.tobytes() and got == want


@pytest.mark.parametrize("lshift,pshift", [(1, 0), (0, 1), (3, 3)])
def test_fused_pack_unaligned_lengths_and_prefix(lshift, pshift):
    """lengths / prefix off 16-byte alignment: scalar block sums and prefix stores"""
    lens, offs, plen = _inputs(300_007, 20, seed=31 + lshift + pshift)
    pool = np.random.default_rng(32).integers(0, 256, plen * 8, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, 8, [(0, 8)], "i32", cap_extra=2, lens_shift=lshift, prefix_shift=pshift)
    pw, want, tw = _expect(lens, offs, pool, 8, [(0, 8)], "i32")
    assert t == tw and p.tobytes() == pw.tobytes() and got == want


def test_fused_pack_many_blocks_per_cta():
    """more records than one 256-sub-tile block per CTA: blocks handed out by ticket"""
    n = 296 * 2 * 262_144 + 12_345  # > (CTAs x max block) on a 148-SM part at 2 CTAs/SM
    rng = np.random.default_rng(33)
    lens = rng.integers(0, 3, n).astype(np.int32)
    offs = np.concatenate([[0], np.cumsum(lens.astype(np.int64))[:-1]]) + 5  # in order, shifted by 5 members
    T = int(lens.sum())
    pool = np.arange(T + 8, dtype=np.uint64)
    p, got, t = _pack(lens, offs, pool.view(np.uint8), 8, [(0, 8)], "i64")
    assert t == T
    assert np.array_equal(p, np.concatenate([[0], np.cumsum(lens.astype(np.int64))]))
    assert np.array_equal(np.frombuffer(got[0], np.uint64), np.arange(5, T + 5, dtype=np.uint64))


@pytest.mark.parametrize("stride,fields", [
    (8, [(0, 4), (4, 4)]),                    # {adc i32, t f32}: 8 staged bytes
    (16, [(8, 8), (0, 4)]),                   # 12 staged bytes, fields out of record order
    (16, [(0, 4), (4, 4), (8, 8)]),           # 16
    (24, [(12, 4), (0, 4), (4, 4), (16, 4)]), # four pools
])
def test_fused_pack_member_field_table(stride, fields):
    """several naturally aligned 4/8-byte member fields scattered into their own pools (SoA scatter):
    8- and 16-byte member records take the fused kernel with record staging and a split drain, the
    24-byte one the two-kernel path"""
    lens, offs, plen = _inputs(400_003, 20, seed=41 + stride + len(fields))
    pool = np.random.default_rng(42).integers(0, 256, plen * stride, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, stride, fields, "i32", cap_extra=9)
    pw, want, tw = _expect(lens, offs, pool, stride, fields, "i32")
    assert t == tw and p.tobytes() == pw.tobytes() and got == want


# ---- invalid segments: reported, never read (lens >= 0, offsets + lens inside the pool) ----

def _pack_raw(lens, offs, pool_members, fields, stride=8, fused=True):
    """sk_jagged_pack on device arrays; returns (total, invalid count)"""
    n = lens.size
    d_lens, d_offs = DeviceArray.from_numpy(lens, CUDA), DeviceArray.from_numpy(offs, CUDA)
    d_pool = DeviceArray(max(pool_members, 1) * stride, np.uint8, CUDA)
    prefix = DeviceArray(n + 1, np.int64 if fused else np.uint16, CUDA)
    cap = 1 << 16
    outs = [DeviceArray(cap * sz, np.uint8, CUDA) for _, sz in fields]
    need = C.c_size_t(0)
    nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
    scratch = DeviceArray(-(-need.value // 256) * 256 + ((cap + 255) // 256 + 1) * 8, np.uint8, CUDA)
    total = DeviceArray(2, np.int64, CUDA)
    nf = len(fields)
    foff = (C.c_int64 * nf)(*[o for o, _ in fields])
    fsz = (C.c_int32 * nf)(*[sz for _, sz in fields])
    dst = (C.c_void_p * nf)(*[o.ptr for o in outs])
    nat.call("sk_jagged_pack", n, d_lens.ptr, TC["i32"], prefix.ptr, TC["i64" if fused else "u16"], d_offs.ptr,
             d_pool.ptr, pool_members, stride, nf, foff, fsz, dst, cap, scratch.ptr, scratch.n, total.ptr,
             nat.stream(0))
    t, bad = (int(v) for v in total.numpy())
    for a in (d_lens, d_offs, d_pool, prefix, scratch, total, *outs):
        a.free()
    return t, bad


@pytest.mark.parametrize("fused", [True, False])
def test_pack_counts_invalid_segments(fused):
    """fused kernel (one 8-byte field) and validate + scan + gather (a 2-byte field) both count records
    whose segment leaves the source pool, and gather nothing for them"""
    n = 50_000
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 5, n).astype(np.int32)
    offs = np.concatenate([[0], np.cumsum(lens.astype(np.int64))[:-1]])
    members = int(lens.sum())
    fields = [(0, 8)] if fused else [(2, 2)]
    assert _pack_raw(lens, offs, members, fields, fused=fused) == (members, 0)
    bad_l, bad_o = lens.copy(), offs.copy()
    bad_l[10] = -1                       # negative length
    i = int(np.flatnonzero(lens)[-1])
    bad_o[i] = members                   # non-empty segment past the end of the pool
    j = int(np.flatnonzero(lens)[0])
    bad_o[j] = -3                        # before its start
    empty = int(np.flatnonzero(lens == 0)[0])
    bad_o[empty] = 1 << 40               # an empty segment's offset is never read: valid
    t, bad = _pack_raw(bad_l, bad_o, members, fields, fused=fused)
    assert bad == 3


def test_collection_pack_rejects_invalid_segments_host_and_device():
    c = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.resize(1000)
    lens, offs, pool = wl.cluster_inputs(1000, seed=4)
    total = jagged.pack(c, "members", lens, offs, pool)

    def state(coll):
        with mc.execution_scope(mc.CUDA):
            return coll.prefix_sums("members").tobytes(), coll.jagged_size("members")

    before = state(c)
    # host inputs: validated before anything is written (strong guarantee)
    for bl, bo in ((np.where(np.arange(1000) == 7, -2, lens), offs), (lens, np.where(lens > 0, offs + pool.size, offs))):
        with pytest.raises(BoundsError):
            jagged.pack(c, "members", bl, bo, pool)
        assert state(c) == before
    # device inputs through the fused kernel: detected on the device, the vector is left empty
    d_pool = DeviceArray.from_numpy(pool, CUDA)
    bad_offs = offs.copy()
    bad_offs[int(np.flatnonzero(lens)[0])] = pool.size
    with pytest.raises(BoundsError):
        jagged.pack(c, "members", DeviceArray.from_numpy(lens, CUDA), DeviceArray.from_numpy(bad_offs, CUDA), d_pool)
    p, size = state(c)
    assert size == 0 and not np.frombuffer(p, np.uint8).any()
    # device inputs on a fresh collection (scan + gather path): validated first, nothing written
    c2 = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c2.resize(1000)
    with pytest.raises(BoundsError):
        jagged.pack(c2, "members", DeviceArray.from_numpy(lens, CUDA), DeviceArray.from_numpy(bad_offs, CUDA), d_pool)
    assert c2.jagged_size("members") == 0
    assert jagged.pack(c, "members", lens, offs, pool) == total


def test_concurrent_fused_packs_on_two_streams():
    """Two full-occupancy packs launched on two streams at once, repeatedly: the fused kernel never waits on a
    CTA that might not be resident (no end-of-grid spin), so they cannot deadlock, and both stay exact."""
    import torch

    n = 2_000_000
    ins = [wl.cluster_inputs(n, seed=s) for s in (21, 22)]
    wants = [_expect_pool(lens, offs, pool) for lens, offs, pool in ins]
    streams = [torch.cuda.Stream(device=0) for _ in range(2)]
    bufs = []
    for lens, offs, pool in ins:
        T = int(lens.astype(np.int64).sum())
        d = [DeviceArray.from_numpy(x, CUDA) for x in (lens, offs, pool)]
        prefix = DeviceArray(n + 1, np.int32, CUDA)
        out = DeviceArray(T, np.uint64, CUDA)
        need = C.c_size_t(0)
        nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
        scratch = DeviceArray(need.value, np.uint8, CUDA)
        total = DeviceArray(2, np.int64, CUDA)
        bufs.append((d, prefix, out, scratch, total, T, pool.size))
    torch.cuda.synchronize()
    for _ in range(20):
        for (d, prefix, out, scratch, total, T, pm), st in zip(bufs, streams):
            foff, fsz, dst = (C.c_int64 * 1)(0), (C.c_int32 * 1)(8), (C.c_void_p * 1)(out.ptr)
            nat.call("sk_jagged_pack", n, d[0].ptr, TC["i32"], prefix.ptr, TC["i32"], d[1].ptr, d[2].ptr, pm, 8, 1,
                     foff, fsz, dst, T, scratch.ptr, scratch.n, total.ptr, st.cuda_stream)
    torch.cuda.synchronize()
    for (d, prefix, out, scratch, total, T, pm), (pw, mw) in zip(bufs, wants):
        assert prefix.numpy().tobytes() == pw.tobytes() and out.numpy().tobytes() == mw.tobytes()
        for a in (*d, prefix, out, scratch, total):
            a.free()


def _expect_pool(lens, offs, pool):
    P = np.concatenate([[0], np.cumsum(lens.astype(np.int64))]).astype(np.int32)
    idx, _ = _gather_index(lens, offs)
    return P, pool[idx]


def test_pack_on_reused_dirty_scratch():
    """The single-field pack zeroes nothing in its scratch between calls (its look-back words and queue
    entries carry a launch generation). One scratch buffer, filled with random bytes first, then reused
    by packs of different sizes, including skewed lengths that take the queue path."""
    rng = np.random.default_rng(31)
    n_max = 1_000_000
    need = C.c_size_t(0)
    nat.call("sk_jagged_scratch_bytes", n_max, C.byref(need))
    scratch = DeviceArray.from_numpy(rng.integers(0, 256, need.value, dtype=np.uint8), CUDA)
    total = DeviceArray(2, np.int64, CUDA)
    cases = [_inputs(n_max, 20, seed=1), _inputs(100_000, 20, seed=2), _skewed_inputs(200_000, seed=5),
             _inputs(n_max, 20, seed=3), _inputs(7, 20, seed=4)]
    try:
        for lens, offs, plen in cases:
            n, T = lens.size, int(lens.astype(np.int64).sum())
            pool = rng.integers(0, 256, plen * 8, dtype=np.uint8)
            d_lens, d_offs, d_pool = (DeviceArray.from_numpy(x, CUDA) for x in (lens, offs, pool))
            prefix = DeviceArray(n + 1, np.int64, CUDA)
            out = DeviceArray(max(T, 1) * 8, np.uint8, CUDA)
            foff, fsz, dst = (C.c_int64 * 1)(0), (C.c_int32 * 1)(8), (C.c_void_p * 1)(out.ptr)
            nat.call("sk_jagged_pack", n, d_lens.ptr, TC["i32"], prefix.ptr, TC["i64"], d_offs.ptr, d_pool.ptr,
                     plen, 8, 1, foff, fsz, dst, T, scratch.ptr, scratch.n, total.ptr, nat.stream(0))
            nat.sync(0)
            pw, want, tw = _expect(lens, offs, pool, 8, [(0, 8)], "i64")
            assert total.numpy().tolist() == [tw, 0]
            assert prefix.numpy().tobytes() == pw.tobytes()
            assert out.numpy()[:T * 8].tobytes() == want[0]
            for a in (d_lens, d_offs, d_pool, prefix, out):
                a.free()
    finally:
        scratch.free()
        total.free()


@pytest.mark.parametrize("stride,field", [(16, (8, 8)), (12, (4, 4)), (24, (16, 8)), (8, (4, 4))])
def test_single_field_of_a_wider_member_record(stride, field):
    """one naturally aligned field out of a wider member record (the register pack's strided loads)"""
    lens, offs, plen = _inputs(300_001, 20, seed=stride + field[0])
    pool = np.random.default_rng(43).integers(0, 256, plen * stride, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, stride, [field], "u32", cap_extra=3)
    pw, want, tw = _expect(lens, offs, pool, stride, [field], "u32")
    assert t == tw and p.tobytes() == pw.tobytes() and got == want


def test_fused_pack_ten_million_records():
    """config 3 at 10M clusters (~100M u64 members, shuffled segments with slack): the whole prefix and
    pool byte-exact against the numpy restatement"""
    lens, offs, plen = _inputs(10_000_000, 20, seed=77)
    pool = np.random.default_rng(78).integers(0, np.iinfo(np.uint64).max, plen, dtype=np.uint64,
                                              endpoint=True).view(np.uint8)
    p, got, t = _pack(lens, offs, pool, 8, [(0, 8)], "i32", cap_extra=1)
    pw, want, tw = _expect(lens, offs, pool, 8, [(0, 8)], "i32")
    assert t == tw and p.tobytes() == pw.tobytes()
    assert got == want


def _tiled_inputs(lens, seed, slack=2):
    rng = np.random.default_rng(seed)
    order = rng.permutation(lens.size)
    gaps = lens[order].astype(np.int64) + rng.integers(0, slack + 1, lens.size)
    offs = np.empty(lens.size, np.int64)
    offs[order] = np.concatenate([[0], np.cumsum(gaps)[:-1]])
    return offs, int(gaps.sum())


@pytest.mark.parametrize("case", ["round_edges", "big_threshold", "tile_edges", "one_huge", "u8_wrap"])
def test_register_pack_structural_edges(case):
    """the register pack's structure: 384-member round boundaries, the 3072-member queueing threshold
    (3072 gathered by the warp, 3073 queued), record counts at tile boundaries, one record holding
    almost every member, and a u8 prefix that wraps"""
    rng = np.random.default_rng(sum(map(ord, case)))
    ptype = "i64"
    if case == "round_edges":  # groups of exactly 383, 384, 385, 767, 768, 769 members
        lens = np.zeros(32 * 6 * 50, np.int32)
        for g, t in enumerate([383, 384, 385, 767, 768, 769] * 50):
            q, r = divmod(t, 32)
            lens[32 * g:32 * g + 32] = q
            lens[32 * g:32 * g + r] += 1
    elif case == "big_threshold":  # groups of 3071, 3072, 3073 and 9000 members among ordinary ones
        lens = rng.integers(0, 21, 40_000).astype(np.int32)
        for g, t in zip((5, 77, 300, 901), (3071, 3072, 3073, 9000)):
            lens[32 * g:32 * g + 32] = t // 32
            lens[32 * g] += t % 32
    elif case == "tile_edges":  # one past / one short of whole 8-warp tiles at several group counts
        lens = rng.integers(0, 21, 256 * 7 * 37 + 1).astype(np.int32)
    elif case == "one_huge":
        lens = rng.integers(0, 3, 50_000).astype(np.int32)
        lens[12_345] = 2_000_000
    else:
        lens = rng.integers(0, 21, 70_001).astype(np.int32)
        ptype = "u8"
    offs, plen = _tiled_inputs(lens, seed=5)
    pool = rng.integers(0, 256, plen * 8, dtype=np.uint8)
    p, got, t = _pack(lens, offs, pool, 8, [(0, 8)], ptype, cap_extra=0 if ptype == "u8" else 7)
    pw, want, tw = _expect(lens, offs, pool, 8, [(0, 8)], ptype)
    assert t == tw and p.tobytes() == pw.tobytes() and got == want


@pytest.mark.parametrize("msize,ptype", [(8, "i64"), (4, "u32")])
def test_scatter_skewed_groups_and_total_bound(msize, ptype):
    """sk_jagged_scatter over a caller prefix with skewed lengths (listed groups gathered by the second
    kernel) and a member bound below the sum: members past `total` are not written"""
    lens, offs, plen = _skewed_inputs(200_000, seed=23)
    pool = np.random.default_rng(24).integers(0, 256, plen * msize, dtype=np.uint8)
    pdt = np.int64 if ptype == "i64" else np.uint32
    P = np.concatenate([[0], np.cumsum(lens.astype(np.int64))]).astype(pdt)
    full = int(P[-1])
    _, want, _ = _expect(lens, offs, pool, msize, [(0, msize)], "i64")
    d_p, d_o, d_pool = (DeviceArray.from_numpy(x, CUDA) for x in (P, offs, pool))
    try:
        for total in (full, full // 2 + 12345):
            out = DeviceArray.from_numpy(np.full(full * msize, 0xAB, np.uint8), CUDA)
            foff, fsz, dst = (C.c_int64 * 1)(0), (C.c_int32 * 1)(msize), (C.c_void_p * 1)(out.ptr)
            nat.call("sk_jagged_scatter", lens.size, d_p.ptr, TC[ptype], d_o.ptr, d_pool.ptr, msize, 1, foff, fsz,
                     dst, total, nat.stream(0))
            nat.sync(0)
            got = out.numpy().tobytes()
            assert got[:total * msize] == want[0][:total * msize]
            assert set(got[total * msize:]) <= {0xAB}
            out.free()
    finally:
        for a in (d_p, d_o, d_pool):
            a.free()
