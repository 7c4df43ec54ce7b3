"""Prepared transfers: copy_collection captured into a CUDA graph and replayed
with one launch (device-resident, pinned-host pipeline, jagged side leaves)."""

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, PINNED, aos_collection, to_host_planes
from oracle import restate as R
from paper_2511_04853_b200 import layouts as ly, sensor, transfer as tr, workloads as wl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("src_ctx", ["cuda", "pinned"])
def test_prepared_transfer_replays_fresh_data(src_ctx):
    n = 200_003
    recs = wl.obj8_records(n, seed=1)
    host = aos_collection(wl.OBJ8_SCHEMA, recs, n, PINNED)
    src = host
    if src_ctx == "cuda":
        src = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
        tr.copy_collection(src, host)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    prep = tr.prepare(dst, src)
    for seed in (2, 3):
        recs = wl.obj8_records(n, seed=seed)
        host.layout._struct_buf._data[: n * 32] = recs.view(np.uint8)
        if src_ctx == "cuda":
            tr.copy_collection(src, host)
        assert prep.run() == "b200-convert"
        planes = to_host_planes(dst)
        want = R.aos_to_planes(recs)
        for i in range(8):
            assert planes[f"f{i}#0"] == want[f"f{i}"][0].tobytes(), (seed, i)
    prep.close()


def test_prepared_transfer_with_jagged_side_leaves_and_staleness():
    rng = np.random.default_rng(4)
    src = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, PINNED)
    src.resize(500)
    src.layout._struct_buf._data[: 500 * 64] = rng.integers(0, 256, 500 * 64, dtype=np.uint8)
    src.jagged_fill("sensors", [rng.integers(0, 99, rng.integers(0, 4), dtype=np.uint64) for _ in range(500)])
    dst = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, CUDA)
    prep = tr.prepare(dst, src)
    prep.run()
    h = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, sk.ContextInfo.host())
    tr.copy_collection(h, dst)
    assert h.dump() == src.dump()
    src.resize(10)
    with pytest.raises(sk.TransferError):
        prep.run()


def test_prepared_transfer_survives_staging_growth():
    """a captured host pipeline references the device staging buffer; a later,
    larger transfer that grows the staging must not free it under the graph"""
    n = 50_000
    recs = wl.obj8_records(n, seed=9)
    small = aos_collection(wl.OBJ8_SCHEMA, recs, n, PINNED)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    prep = tr.prepare(dst, small)
    big_n = 40_000_000  # 1.28 GB: several full pipeline chunks, grows the staging
    big = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, PINNED)
    big.resize(big_n)
    big_dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(big_dst, big)
    big.free()
    big_dst.free()
    recs2 = wl.obj8_records(n, seed=10)
    small.layout._struct_buf._data[: n * 32] = recs2.view(np.uint8)
    prep.run()
    planes = to_host_planes(dst)
    want = R.aos_to_planes(recs2)
    for i in range(8):
        assert planes[f"f{i}#0"] == want[f"f{i}"][0].tobytes()
    prep.close()


def test_prepare_refuses_host_only_pairs():
    """pinned <-> pinned copies run on the host, outside the graph; a prepared transfer over them
    would replay nothing (bulk / plane copies) or stale side data (Particle's jagged pools)."""
    src = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, PINNED)
    src.resize(10)
    for kind in (ly.PER_FIELD, ly.AOS):
        dst = sk.Collection(sensor.PARTICLE_SCHEMA, kind, PINNED)
        with pytest.raises(sk.TransferError):
            tr.prepare(dst, src)
