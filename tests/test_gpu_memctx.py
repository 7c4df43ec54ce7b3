"""The cuda / pinned memory contexts: copier matrix, device memmove contract
(C5, test_acceptance.py:558-583), device-side size changes, migration."""

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, HOST, PINNED
from paper_2511_04853_b200 import layouts as ly
from paper_2511_04853_b200 import memctx as mc
from paper_2511_04853_b200 import sensor, transfer as tr

pytestmark = pytest.mark.gpu


def test_copier_matrix_round_trips():
    pattern = np.random.default_rng(1).integers(0, 256, 4096, dtype=np.uint8)
    infos = [HOST, PINNED, CUDA]
    for a in infos:
        for b in infos:
            src = mc.allocate(HOST, 4096)
            src._data[:] = pattern
            x = mc.allocate(a, 4096)
            y = mc.allocate(b, 4096)
            mc.memcopy_with_context(x, 0, src, 0, 4096)
            mc.memcopy_with_context(y, 100, x, 0, 3000)
            out = mc.allocate(HOST, 4096)
            out._data[:] = 0
            mc.memcopy_with_context(out, 0, y, 100, 3000)
            assert np.array_equal(out._data[:3000], pattern[:3000]), (a, b)
            for buf in (src, x, y, out):
                mc.deallocate(buf)


def test_device_memmove_overlap_oracle():
    """Exhaustive same-buffer copies on a 48-byte device buffer vs copy-via-temp."""
    size = 48
    buf = mc.allocate(CUDA, size)
    stage = mc.allocate(PINNED, size)
    base = np.arange(size, dtype=np.uint8)
    bad = 0
    for count in range(0, size + 1, 3):
        for s in range(size + 1 - count):
            for d in range(size + 1 - count):
                stage._data[:] = base
                mc.memcopy_with_context(buf, 0, stage, 0, size)
                mc.memcopy_with_context(buf, d, buf, s, count)
                mc.memcopy_with_context(stage, 0, buf, 0, size)
                exp = base.copy()
                exp[d : d + count] = base[s : s + count]
                bad += not np.array_equal(stage._data, exp)
    assert bad == 0


def test_device_resize_insert_erase_match_host():
    rng = np.random.default_rng(2)
    host = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, HOST)
    dev = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, CUDA)
    host.resize(20)
    host.column("energy").np[:] = rng.standard_normal(20).astype(np.float32)
    host.column("noisy_count").np[:] = rng.integers(0, 255, (4, 20))
    host.jagged_fill("sensors", [rng.integers(0, 99, rng.integers(0, 4), dtype=np.uint64) for _ in range(20)])
    tr.copy_collection(dev, host)
    for c, scope in ((host, mc.HOST), (dev, mc.CUDA)):
        with mc.execution_scope(scope):
            c.insert_records(3, 5)
            c.erase_records(10, 4)
            c.jagged_resize("sensors", 2, 7)
            c.resize(30)
            c.resize(25)
    back = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, HOST)
    tr.copy_collection(back, dev)
    assert back.dump() == host.dump()


def test_device_collection_refuses_host_scope_access():
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    with pytest.raises(sk.NotResizableError):
        dev.resize(3)
    with mc.execution_scope(mc.CUDA):
        dev.resize(3)
    with pytest.raises(sk.AccessError):
        dev.column("energy").read()
    with mc.execution_scope(mc.CUDA), pytest.raises(sk.AccessError):
        dev.column("energy").np


def test_migration_round_trip_keeps_contents():
    c = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, HOST)
    c.resize(11)
    c.column("origin").np[:] = np.arange(11, dtype=np.uint64) * 3
    c.jagged_fill("sensors", [[i] * (i % 3) for i in range(11)])
    ref = c.dump()
    for info in (CUDA, PINNED, CUDA, HOST):
        c.update_memory_context_info(info)
    assert c.dump() == ref


@pytest.mark.parametrize("nops", [1, 7, 300])
def test_copy_rows_batched_moves_and_fills_vs_numpy(nops):
    """memctx.copy_rows -> sk_move_batch_async: random self-overlapping moves and zero fills over many
    buffers (300 ops crosses the 128-op batch), every move reading its source before any fill lands; the
    same ops applied to host twins with numpy are the oracle."""
    rng = np.random.default_rng(nops)
    nbuf = min(nops, 40)
    sizes = rng.integers(64, 200_000, nbuf)
    dev = [mc.allocate(CUDA, int(n)) for n in sizes]
    host = [mc.allocate(HOST, int(n)) for n in sizes]
    for d, h in zip(dev, host):
        h._data[:] = rng.integers(0, 256, h.length_bytes, dtype=np.uint8)
        mc.memcopy_with_context(d, 0, h, 0, h.length_bytes)
    # disjoint destinations per buffer: split each buffer into slices, one op per slice
    ops_d, ops_h = [], []
    per = max(1, nops // nbuf)
    for b in range(nbuf):
        cuts = np.sort(rng.choice(np.arange(1, sizes[b]), size=min(per * 2, sizes[b] - 1), replace=False))
        edges = [0, *cuts.tolist(), int(sizes[b])]
        for lo, hi in zip(edges[::2], edges[1::2]):
            n = hi - lo
            if n <= 0 or len(ops_d) >= nops:
                continue
            if rng.random() < 0.3:
                ops_d.append(mc.RowOp(dev[b], lo, None, 0, n))
                ops_h.append(mc.RowOp(host[b], lo, None, 0, n))
            else:
                src = int(rng.integers(0, sizes[b] - n + 1))  # may overlap its own destination
                ops_d.append(mc.RowOp(dev[b], lo, dev[b], src, n))
                ops_h.append(mc.RowOp(host[b], lo, host[b], src, n))
    mc.copy_rows(ops_d)
    mc.copy_rows(ops_h)
    for d, h in zip(dev, host):
        out = mc.allocate(HOST, d.length_bytes)
        mc.memcopy_with_context(out, 0, d, 0, d.length_bytes)
        assert np.array_equal(out._data, h._data)
        mc.deallocate(out)
    for buf in dev + host:
        mc.deallocate(buf)


def test_large_pageable_buffers_are_pinned_once_and_released():
    """memctx.pin_for_transfer: a >= 8 MB pageable host buffer taking part in a device copy is page-locked
    once; deallocation (or garbage collection) unregisters it."""
    import weakref

    n = 16 << 20
    host = mc.allocate(HOST, n)
    host._data[:] = 7
    dev = mc.allocate(CUDA, n)
    mc.memcopy_with_context(dev, 0, host, 0, n)
    assert isinstance(host._keep, weakref.finalize) and host._keep.alive
    fin = host._keep
    mc.memcopy_with_context(host, 0, dev, 0, n)  # reused, not registered twice
    assert host._keep is fin
    mc.deallocate(host)
    assert not fin.alive
    small = mc.allocate(HOST, 4096)
    mc.memcopy_with_context(small, 0, dev, 0, 4096)
    assert small._keep is None  # below the threshold: stays pageable
    for b in (small, dev):
        mc.deallocate(b)


def test_host_return_arrays_are_pinned_and_recycled():
    """host_return_array: page-locked, reused only once every array viewing the buffer is gone"""
    import gc

    import numpy as np

    from paper_2511_04853_b200 import _native as nat
    from paper_2511_04853_b200 import memctx as mc

    small = mc.host_return_array(16, np.float32)
    assert small.size == 16  # below RETURN_POOL_MIN: a plain array
    n = 3_000_000
    a = mc.host_return_array(n, np.float32)
    a[:] = np.arange(n, dtype=np.float32)
    view = a[10:20]
    p0 = a.ctypes.data
    del a
    gc.collect()
    b = mc.host_return_array(n, np.float32)
    pb = b.ctypes.data
    assert pb != p0  # the view still holds the first buffer
    assert view.tolist() == list(range(10, 20))
    del view, b
    gc.collect()
    c = mc.host_return_array(n, np.float32)
    assert c.ctypes.data in (p0, pb)  # recycled from the pool
    # a device -> host copy into it lands at full speed and intact
    d = nat.malloc(0, n * 4)
    try:
        nat.memset(d, 0x3F, n * 4, 0)
        nat.memcpy(c.ctypes.data, d, n * 4, 0)
        nat.sync(0)
        assert (c.view(np.uint32) == 0x3F3F3F3F).all()
    finally:
        nat.free(0, d)
