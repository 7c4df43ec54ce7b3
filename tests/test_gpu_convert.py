"""Parity of the conversion engine (K1/K2/K3) against the reference's golden
vectors and the oracle, through the public API and the C-ABI."""

import itertools

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, HOST, PINNED, aos_collection, device_bytes_equal, device_to_numpy, to_host_aos, to_host_planes
from oracle import restate as R
from paper_2511_04853_b200 import convert as cv
from paper_2511_04853_b200 import layouts as ly
from paper_2511_04853_b200 import memctx as mc
from paper_2511_04853_b200 import schema as sc
from paper_2511_04853_b200 import sensor, transfer as tr, workloads as wl
from skhelp import golden

pytestmark = pytest.mark.gpu

CTX = {"host": HOST, "pinned": PINNED, "cuda": CUDA}


def obj8_golden():
    g = golden("obj8.npz")
    return g, int(g["n"])


@pytest.mark.parametrize("src_ctx", ["host", "pinned", "cuda"])
@pytest.mark.parametrize("dst_kind", [ly.PER_FIELD, ly.ARENA])
def test_obj8_aos_to_planes_bit_exact_vs_reference(src_ctx, dst_kind):
    g, n = obj8_golden()
    src = aos_collection(wl.OBJ8_SCHEMA, g["aos"], n, HOST)
    if src_ctx != "host":
        moved = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CTX[src_ctx])
        assert tr.copy_collection(moved, src) == "bulk-same-kind"
        src = moved
    arena = ly.ArenaSpec({sc.MAIN_TAG: n + 3}) if dst_kind == ly.ARENA else None
    dst = sk.Collection(wl.OBJ8_SCHEMA, dst_kind, CUDA, arena)
    assert tr.copy_collection(dst, src) == "b200-convert"
    planes = to_host_planes(dst)
    for i in range(8):
        assert planes[f"f{i}#0"] == g[f"plane:f{i}#0"].tobytes(), i


@pytest.mark.parametrize("dst_ctx", ["host", "pinned", "cuda"])
def test_obj8_planes_to_aos_bit_exact(dst_ctx):
    g, n = obj8_golden()
    src = aos_collection(wl.OBJ8_SCHEMA, g["aos"], n, HOST)
    dev_planes = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(dev_planes, src)
    back = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CTX[dst_ctx])
    assert tr.copy_collection(back, dev_planes) == "b200-convert"
    assert to_host_aos(back).tobytes() == g["aos"].tobytes()


def test_particle_multislot_and_jagged_side_leaves_vs_reference():
    g = golden("particle.npz")
    n = int(g["n"])
    src = aos_collection(sensor.PARTICLE_SCHEMA, g["aos"], n, HOST)
    # jagged side leaves: rebuild the reference's pool + prefix through the public API
    pool = g["plane:sensors.value#0"].view(np.uint64)
    prefix = g["plane:sensors.prefix_sum#0"].view(np.int32)
    segs = [pool[prefix[i]:prefix[i + 1]] for i in range(n)]
    src.jagged_fill("sensors", segs)
    for kind, arena in ((ly.PER_FIELD, None), (ly.ARENA, ly.ArenaSpec({sc.MAIN_TAG: n + 7, "sensors": 6000}, 64))):
        dst = sk.Collection(sensor.PARTICLE_SCHEMA, kind, CUDA, arena)
        assert tr.copy_collection(dst, src) == "b200-convert"
        planes = to_host_planes(dst)
        for key, val in g.items():
            if key.startswith("plane:"):
                assert planes[key[6:]] == val.tobytes(), key
        if kind == ly.ARENA:
            img = device_to_numpy(dst.layout._buf.ptr, dst.layout.total_bytes)
            ref = g["arena_image"]
            # the reference arena image: every leaf region up to its size matches
            for lf in dst.plan.leaves:
                off = dst.layout.leaf_offset(lf)
                ln = dst.layout.plane_len(lf) * lf.value_type.size_bytes
                for k in range(lf.extent_multiplier):
                    o = off + k * dst.layout._cap_len(lf) * lf.value_type.size_bytes
                    assert img[o:o + ln].tobytes() == ref[o:o + ln].tobytes(), lf.dotted


def _random_particles(n, seed):
    rng = np.random.default_rng(seed)
    c = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, HOST)
    c.resize(n)
    c.layout._struct_buf._data[: n * 64] = rng.integers(0, 256, n * 64, dtype=np.uint8)
    c.jagged_fill("sensors", [rng.integers(0, 2**63, rng.integers(0, 5), dtype=np.uint64) for _ in range(n)])
    return c


KINDS = [ly.PER_FIELD, ly.ARENA, ly.AOS]


def _make(kind, ctx, n, total):
    arena = ly.ArenaSpec({sc.MAIN_TAG: n + 5, "sensors": total + 9}) if kind == ly.ARENA else None
    return sk.Collection(sensor.PARTICLE_SCHEMA, kind, CTX[ctx], arena)


def test_transfer_matrix_every_pair_round_trips():
    """C4 (test_acceptance.py:504-552) widened: 9 endpoints^2 = 81 ordered pairs,
    all dump-identical; the reference's 4 unsupported pairs (AoS destination
    off-host) are served by K2 here."""
    n = 37
    base = _random_particles(n, 5)
    ref = base.dump()
    total = base.jagged_size("sensors")
    eps = list(itertools.product(KINDS, ["host", "pinned", "cuda"]))
    for (k1, c1), (k2, c2) in itertools.product(eps, eps):
        a = _make(k1, c1, n, total)
        tr.copy_collection(a, base)
        b = _make(k2, c2, n, total)
        tr.copy_collection(b, a)
        h = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, HOST)
        tr.copy_collection(h, b)
        assert h.dump() == ref, (k1, c1, k2, c2)
        for c in (a, b, h):
            c.free()


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 255, 511, 513, 4099, 100003])
def test_obj8_tail_sizes_vs_oracle(n):
    recs = wl.obj8_records(n, seed=n)
    src = aos_collection(wl.OBJ8_SCHEMA, recs, n, PINNED)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(dst, src)
    planes = to_host_planes(dst)
    want = R.aos_to_planes(recs)
    for i in range(8):
        assert planes[f"f{i}#0"] == want[f"f{i}"][0].tobytes()
    back = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
    tr.copy_collection(back, dst)
    assert to_host_aos(back).tobytes() == recs.tobytes()


def test_unaligned_plane_pitch_uses_safe_path():
    # capacity 5 -> multi-slot planes at 20-byte pitch: not 16-byte aligned
    src = _random_particles(5, 9)
    dst = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        dst.reserve(5)
    tr.copy_collection(dst, src)
    assert dst.capacity() == 5
    h = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, HOST)
    tr.copy_collection(h, dst)
    assert h.dump() == src.dump()
    back = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, CUDA)
    tr.copy_collection(back, dst)
    assert to_host_aos(back).tobytes() == np.array(src.layout._struct_buf._data[: 5 * 64]).tobytes()


def test_one_million_obj8_pinned_h2d_vs_oracle():
    n = 1_000_000
    recs = wl.obj8_records(n)
    src = aos_collection(wl.OBJ8_SCHEMA, recs, n, PINNED)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    assert tr.copy_collection(dst, src) == "b200-convert"
    planes = to_host_planes(dst)
    want = R.aos_to_planes(recs)
    for i in range(8):
        assert planes[f"f{i}#0"] == want[f"f{i}"][0].tobytes()


def test_hundred_million_round_trip_on_device():
    """Size-independent property at the config-4/5 scale: AoS -> planes -> AoS
    is the identity on 3.2 GB of random records; a 1M-record sample of the
    planes also matches the oracle."""
    n = 100_000_000
    src = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
    with mc.execution_scope(mc.CUDA):
        src.reserve(n)
    with src.layout.engine_ops():
        src.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    wl.fill_random_device(src.layout._struct_buf.ptr, n * 32, seed=77, device=0)
    planes = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(planes, src)
    back = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
    tr.copy_collection(back, planes)
    assert device_bytes_equal(src.layout._struct_buf.ptr, back.layout._struct_buf.ptr, n * 32)
    lo = n - 1_000_000
    raw = device_to_numpy(src.layout._struct_buf.ptr + lo * 32, 1_000_000 * 32)
    want = R.aos_to_planes(raw.view(wl.OBJ8_AOS_DTYPE))
    for i in range(8):
        got = device_to_numpy(planes.layout.plane_address(planes.plan.leaf(f"f{i}")) + lo * 4, 4_000_000)
        assert got.tobytes() == want[f"f{i}"][0].tobytes()
    for c in (src, planes, back):
        c.free()


def test_past_four_gib_offsets_vs_oracle():
    """160M Obj8 records = 5.12 GB of AoS: tiles whose AoS byte offsets lie
    past 2^32 (and the last record) are checked against the oracle's
    restatement of the splitmix input image, both directions (K1 and K2)."""
    n, seed = 160_000_000, 31
    src = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
    with mc.execution_scope(mc.CUDA):
        src.reserve(n)
    with src.layout.engine_ops():
        src.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    wl.fill_random_device(src.layout._struct_buf.ptr, n * 32, seed=seed, device=0)
    planes = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(planes, src)
    t = 8192
    first_past = (1 << 32) // 32
    starts = [first_past - t // 2, first_past, 150_000_000, n - t]
    for r0 in starts:
        want = R.splitmix_image(seed, 0, r0 * 32, t * 32).view(wl.OBJ8_AOS_DTYPE)
        for i in range(8):
            got = device_to_numpy(planes.layout.plane_address(planes.plan.leaf(f"f{i}")) + r0 * 4, t * 4)
            assert got.tobytes() == np.ascontiguousarray(want[f"f{i}"]).tobytes(), (r0, i)
    back = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
    tr.copy_collection(back, planes)
    for r0 in starts:
        got = device_to_numpy(back.layout._struct_buf.ptr + r0 * 32, t * 32)
        assert got.tobytes() == R.splitmix_image(seed, 0, r0 * 32, t * 32).tobytes(), r0
    assert device_bytes_equal(src.layout._struct_buf.ptr, back.layout._struct_buf.ptr, n * 32)
    for c in (src, planes, back):
        c.free()


TRACK_FIELDS = [("pz", "f32"), ("px", "f32"), ("x", "f32"), ("charge", "i32")]


@pytest.mark.parametrize("lanes", [32, 64, 128])
@pytest.mark.parametrize("src_kind", [ly.AOS, ly.PER_FIELD])
def test_aosoa_subset_reorder_cast_vs_oracle(lanes, src_kind):
    n = 100_003
    recs = wl.track_records(n)
    host = aos_collection(wl.TRACK_SCHEMA, recs, n, PINNED)
    src = sk.Collection(wl.TRACK_SCHEMA, src_kind, CUDA)
    tr.copy_collection(src, host)
    fields = [sk.AosoaField(leaf, dt) for leaf, dt in TRACK_FIELDS]
    a = sk.to_aosoa(src, fields, lanes)
    want = R.to_aosoa(recs, TRACK_FIELDS, lanes, a.tile_bytes)
    got = a.to_host_bytes()
    assert got.tobytes() == want
    # identity-typed field survives the round trip back into a collection
    back = sk.Collection(wl.TRACK_SCHEMA, ly.PER_FIELD, CUDA)
    sk.from_aosoa(a, back)
    with mc.execution_scope(mc.CUDA):
        assert np.array_equal(back.column("charge").read(), recs["charge"])
    a.free()


CAST_CASES = [("f64", "f32"), ("f32", "f64"), ("i32", "i64"), ("i64", "i32"), ("u8", "u32"), ("u64", "f32"),
              ("i64", "f64"), ("i32", "f32"), ("u16", "u8"), ("f64", "bool"), ("i32", "u16")]


@pytest.mark.parametrize("st,dt", CAST_CASES)
def test_cast_semantics_match_numpy_astype(st, dt):
    rng = np.random.default_rng(3)
    npt = {"f64": np.float64, "f32": np.float32, "i32": np.int32, "i64": np.int64, "u8": np.uint8, "u16": np.uint16,
           "u32": np.uint32, "u64": np.uint64, "bool": np.bool_}
    n = 4096
    raw = rng.integers(0, 256, n * np.dtype(npt[st]).itemsize, dtype=np.uint8)
    vals = raw.view(npt[st]).copy()
    if st == "f64":
        vals[:8] = [3.5e38, 7e-46, 1.0 + 2.0 ** -24, np.inf, -0.0, 2.0 ** -150, 1e300, -1e-300]
        vals.view(np.uint64)[8:12] = [0x7FF8DEAD00000000, 0xFFF0000000000001, 0x7FF4000000000000, 0x7FFFFFFFFFFFFFFF]
    schema = sc.Schema("C", (sc.declare_per_item("v", sc.ScalarType(st)),))
    host = sk.Collection(schema, ly.PER_FIELD, HOST)
    host.resize(n)
    host.column("v").np[:] = vals
    dev = sk.Collection(schema, ly.PER_FIELD, CUDA)
    tr.copy_collection(dev, host)
    a = sk.to_aosoa(dev, [sk.AosoaField("v", dt)], 128)
    with np.errstate(all="ignore"):
        want = vals.astype(npt[dt])
    got = a.to_host_bytes()[: n * want.itemsize].view(npt[dt])
    assert got.tobytes() == want.tobytes()


def test_capacity_error_before_any_write():
    g, n = obj8_golden()
    src = aos_collection(wl.OBJ8_SCHEMA, g["aos"], n, HOST)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.ARENA, CUDA, ly.ArenaSpec({sc.MAIN_TAG: 10}))
    with pytest.raises(sk.CapacityError):
        tr.copy_collection(dst, src)
    assert dst.size() == 0


def test_device_oom_maps_to_allocation_error_with_rollback():
    c = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, HOST)
    c.resize(1000)
    c.column("f1").np[:] = np.arange(1000, dtype=np.int32)
    mc.configure_cuda(capacity_bytes=1000)
    try:
        with pytest.raises(sk.AllocationError):
            c.update_memory_context_info(CUDA)
        assert c.info == HOST and np.array_equal(c.column("f1").read(), np.arange(1000, dtype=np.int32))
    finally:
        mc.configure_cuda(None)
    c.update_memory_context_info(CUDA)
    c.update_memory_context_info(PINNED)
    assert np.array_equal(c.column("f1").read(), np.arange(1000, dtype=np.int32))


def test_async_copy_then_sync():
    g, n = obj8_golden()
    src = aos_collection(wl.OBJ8_SCHEMA, g["aos"], n, PINNED)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(dst, src, {"async": True})
    from paper_2511_04853_b200 import _native as nat
    nat.sync(0)
    assert to_host_planes(dst)["f3#0"] == g["plane:f3#0"].tobytes()


def test_engine_uses_tma_bulk_path_for_aligned_collections():
    n = 1 << 20
    src = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    for c in (src, dst):
        with mc.execution_scope(mc.CUDA):
            c.reserve(n)
    info = cv.plan_info(cv.plan_desc(dst.layout, src.layout, n))
    assert info["bulk_in"] and info["bulk_out"] and info["mode"] == 1


@pytest.mark.parametrize("back_kind", [ly.PER_FIELD, ly.AOS])
@pytest.mark.parametrize("lanes", [4, 32, 64])
def test_aosoa_to_planes_all_fields_vs_records(lanes, back_kind):
    """AoSoA -> per_field (the block transform) and AoSoA -> AoS (the record-group transform reading AoSoA
    blocks): identity fields come back bit-exact, f64 fields stored as f32 come back as f64(f32(x))
    (numpy astype both ways)"""
    n = 50_001
    recs = wl.track_records(n)
    host = aos_collection(wl.TRACK_SCHEMA, recs, n, PINNED)
    src = sk.Collection(wl.TRACK_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(src, host)
    names = list(recs.dtype.names)
    code = {"charge": "i32", "id": "u64"}
    fields = [sk.AosoaField(nm, "f32" if nm in ("px", "py") else code.get(nm, "f64")) for nm in names]
    a = sk.to_aosoa(src, fields, lanes)
    back = sk.Collection(wl.TRACK_SCHEMA, back_kind, CUDA)
    sk.from_aosoa(a, back)
    with mc.execution_scope(mc.CUDA):
        for nm in names:
            got = back.column(nm).read()
            want = recs[nm]
            if nm in ("px", "py"):
                with np.errstate(all="ignore"):
                    want = want.astype(np.float32).astype(np.float64)
            assert got.tobytes() == np.ascontiguousarray(want).tobytes(), nm
    a.free()


def test_from_aosoa_grows_through_resize():
    """records created by from_aosoa start at zero in the leaves the AoSoA does not carry, and a
    jagged vector's prefix sums stay monotone (all records empty)."""
    n = 10_007
    parts = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        parts.resize(5)
    src = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        src.resize(n)
    fields = [sk.AosoaField("energy", "f32"), sk.AosoaField("origin", "u64")]
    a = sk.to_aosoa(src, fields, 64)
    sk.from_aosoa(a, parts)
    with mc.execution_scope(mc.CUDA):
        assert parts.size() == n
        assert not parts.prefix_sums("sensors").any()
        assert parts.jagged_size("sensors") == 0
        assert not parts.column("x_variance").read().any()
        assert not parts.column("noisy_count").read().any()
    a.free()
