"""Host-side logic (no GPU): plans, byte geometry, registries, descriptors, ABI."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat
from paper_2511_04853_b200 import convert as cv
from paper_2511_04853_b200 import layouts as ly
from paper_2511_04853_b200 import memctx as mc
from paper_2511_04853_b200 import schema as sc
from paper_2511_04853_b200 import sensor, shard, transfer as tr, workloads as wl
from skhelp import ROOT, golden


def _leaf_sig(plan):
    return [f"{lf.dotted}|{lf.value_type.np_dtype.str}|{lf.size_tag}|{lf.extent_multiplier}|{lf.role}"
            for lf in plan.leaves]


def test_flatten_matches_reference_plans():
    g = golden("geometry.npz")
    assert _leaf_sig(sensor.PARTICLE_PLAN) == list(g["particle_leaves"])
    assert _leaf_sig(sensor.SENSOR_PLAN) == list(g["sensor_leaves"])


def test_record_strides_match_reference():
    g = golden("geometry.npz")
    for schema, key in ((sensor.PARTICLE_SCHEMA, "particle_stride"), (sensor.SENSOR_SCHEMA, "sensor_stride")):
        lay = ly.build_layout(ly.AOS, sc.flatten(schema))
        assert lay.record_stride == int(g[key])
        lay.free()
    assert ly.build_layout(ly.AOS, sc.flatten(wl.OBJ8_SCHEMA)).record_stride == 32
    assert ly.build_layout(ly.AOS, sc.flatten(wl.TRACK_SCHEMA)).record_stride == 60


def test_sensor_struct_dtype_is_the_handwritten_aos_image():
    lay = ly.build_layout(ly.AOS, sensor.SENSOR_PLAN)
    offs = lay.struct_offsets
    assert [offs[k] for k in ("type", "counts", "energy", "calibration_data.noisy",
                              "calibration_data.parameter_A", "calibration_data.noise_B")] == [0, 1, 9, 13, 14, 26]
    assert sensor.SENSOR_AOS_DTYPE.itemsize == 30


@pytest.mark.parametrize("align", [16, 64, 4096])
def test_arena_offsets_match_reference(align):
    g = golden("geometry.npz")
    lay = ly.build_layout(ly.ARENA, sensor.PARTICLE_PLAN, None, ly.ArenaSpec({sc.MAIN_TAG: 10, "sensors": 33}, align))
    assert [lay.leaf_offset(lf) for lf in sensor.PARTICLE_PLAN.leaves] == list(g[f"arena_offsets_{align}"])
    assert lay.total_bytes == int(g[f"arena_total_{align}"])
    assert all(lay.leaf_offset(lf) % align == 0 for lf in sensor.PARTICLE_PLAN.leaves)


def test_growth_policy_matches_reference():
    g = golden("geometry.npz")
    lay = ly.build_layout(ly.PER_FIELD, sensor.PARTICLE_PLAN)
    caps = []
    for n in (1, 5, 17):
        lay.resize(sc.MAIN_TAG, n)
        caps.append(lay.capacity(sc.MAIN_TAG))
    assert caps == list(g["growth"]) == [4, 8, 17]


def test_per_field_slot_planes_at_capacity_pitch():
    c = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD)
    c.resize(6)
    lay = c.layout
    leaf = c.plan.leaf("E_contribution.value")
    assert lay.plane_address(leaf, 2) - lay.plane_address(leaf, 0) == 2 * lay.capacity() * 4
    for flat in range(24):
        lay.write_element(leaf, flat, np.float32(flat * 0.5))
    col = lay.column_np(leaf)
    assert col[3, 5] == np.float32((3 * 6 + 5) * 0.5)


def test_plan_desc_aos_to_planes_fields():
    src = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS)
    dst = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD)
    for c in (src, dst):
        c.resize(9)
    d = cv.plan_desc(dst.layout, src.layout, 9)
    assert d.src_kind == nat.KIND_AOS and d.dst_kind == nat.KIND_PLANES
    assert d.src_stride == 64 and d.nfields == 6 + 4 + 4 + 4
    offs = [d.fields[i].src_off for i in range(d.nfields)]
    assert offs[:6] == [0, 4, 8, 12, 20, 24] and offs[6:10] == [28, 32, 36, 40] and offs[-4:] == [60, 61, 62, 63]
    leaf = dst.plan.leaf("noisy_count.value")
    assert d.fields[d.nfields - 1].dst_plane == dst.layout.plane_address(leaf, 3)
    assert d.fields[3].src_type == nat.TYPE_CODES["u64"]


def test_host_memmove_contract_exhaustive_small():
    # the C5 overlap oracle (test_acceptance.py:558-583) on the host copier, n=24
    buf = mc.allocate(mc.ContextInfo.host(), 24)
    base = np.arange(24, dtype=np.uint8)
    for count in range(25):
        for s in range(25 - count):
            for d in range(25 - count):
                buf._data[:] = base
                mc.memcopy_with_context(buf, d, buf, s, count)
                exp = base.copy()
                exp[d : d + count] = base[s : s + count]
                assert np.array_equal(buf._data, exp)
    mc.deallocate(buf)


def test_memcopy_validation_errors():
    a = mc.allocate(mc.ContextInfo.host(), 8)
    b = mc.allocate(mc.ContextInfo.host(), 8)
    with pytest.raises(sk.CopyError):
        mc.memcopy_with_context(a, 0, b, 4, 8)
    with pytest.raises(sk.CopyError):
        mc.memcopy_with_context(a, 0, b, 0, 4, {"stream": 3})  # test_memctx.py:139-146
    mc.deallocate(b)
    with pytest.raises(sk.BufferStateError):
        mc.memcopy_with_context(a, 0, b, 0, 4)
    with pytest.raises(sk.BufferStateError):
        mc.deallocate(b)
    mc.deallocate(a)


def test_cuda_context_params_and_guards():
    ctx = mc.get_context(mc.CUDA)
    ctx.validate_params({"device_id": 1})
    for bad in ({"device_id": -1}, {"device_id": "0"}, {"stream": 1}):
        with pytest.raises(sk.MemoryContextError):
            ctx.validate_params(bad)
    assert ctx.device_of({"device_id": 3}) == 3
    assert not ctx.host_visible and mc.get_context(mc.PINNED).host_visible


def test_registry_order_and_choice_predicates():
    assert tr.registered_transfers()[:3] == ("b200-convert", "bulk-same-kind", "plane-copy")
    with pytest.raises(sk.RegistryError):
        tr.register_transfer("bulk-same-kind", tr.TransferPriority.SAME_LAYOUT_KIND, lambda d, s: False, None)
    a = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS)
    p = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD)
    r = sk.Collection(wl.OBJ8_SCHEMA, ly.ARENA, None, ly.ArenaSpec({sc.MAIN_TAG: 16}))
    assert tr._convert_applies(p, a) and tr._convert_applies(a, p)
    assert not tr._convert_applies(p, r) and tr._planes_applies(p, r) and tr._planes_applies(r, p)
    assert tr._bulk_applies(a, sk.Collection(wl.OBJ8_SCHEMA, ly.AOS))


def test_copy_collection_rejects_alias_and_mismatch():
    a = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD)
    with pytest.raises(sk.TransferError):
        tr.copy_collection(a, a)
    with pytest.raises(sk.SchemaMismatchError):
        tr.copy_collection(sk.Collection(wl.TRACK_SCHEMA), a)


def test_same_kind_host_transfer_is_bulk_and_exact():
    src = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD)
    src.resize(50)
    src.column("f0").np[:] = np.arange(50, dtype=np.float32)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD)
    assert tr.copy_collection(dst, src) == "bulk-same-kind"
    assert np.array_equal(dst.column("f0").read(), np.arange(50, dtype=np.float32))
    r = sk.Collection(wl.OBJ8_SCHEMA, ly.ARENA, None, ly.ArenaSpec({sc.MAIN_TAG: 64}))
    assert tr.copy_collection(r, src) == "plane-copy"
    assert r.dump() == src.dump()


def test_device_collection_guards_from_host_scope():
    # mockdev semantics (memctx.py:386-395): device elements are not touchable from host code
    c = sk.Collection.__new__(sk.Collection)
    lay = ly.LayoutInstance.__new__(ly.LayoutInstance)
    lay.info = mc.ContextInfo.cuda(0)
    lay.capabilities = ly.LayoutInstance._build_capabilities(lay)
    assert lay.capabilities.flags("host") == ly.AccessFlags()
    assert lay.capabilities.flags("cuda").resizable


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 1000, 10**9):
        for world in (1, 2, 3, 8):
            spans = [shard.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    assert shard.exclusive_offsets([3, 0, 5, 2]) == [0, 3, 3, 8]


# ---- record-signature specialisation (NVRTC, compiled here without a GPU) -------------------

def _spec_check(desc, epi=None):
    buf = ctypes.create_string_buffer(1 << 17)
    ln = ctypes.c_size_t()
    ep = (ctypes.c_int * 7)(*epi) if epi else None
    st = nat.lib().sk_convert_specialize_check(ctypes.byref(desc), ep, buf, len(buf), ctypes.byref(ln))
    return st, buf.value.decode(), nat.lib().sk_last_error().decode()


def test_specialised_transforms_compile_for_sm100a():
    a = sk.Collection(sensor.SENSOR_SCHEMA, ly.AOS)
    p = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD)
    for c in (a, p):
        c.resize(777)
    st, src, err = _spec_check(cv.plan_desc(p.layout, a.layout, 777))
    assert st == nat.SK_OK, err
    assert "const uint32_t W14 = w[14];" in src and "kFusedEpilogue = false" in src  # 2 x 30 B = 15 words
    names = [lf.dotted for lf, _ in cv.main_slots(a.layout)]
    epi = [names.index(k) for k in ("counts", "energy", "calibration_data.noisy", "calibration_data.parameter_A",
                                    "calibration_data.parameter_B", "calibration_data.noise_A",
                                    "calibration_data.noise_B")]
    st, src, err = _spec_check(cv.plan_desc(p.layout, a.layout, 777), epi)
    assert st == nat.SK_OK and "sensor_noise" in src, err
    # planes -> AoS of the 64 B Particle record (u8 slots force the element path)
    pa = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS)
    pp = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD)
    for c in (pa, pp):
        c.resize(300)
    st, src, err = _spec_check(cv.plan_desc(pa.layout, pp.layout, 300))
    assert st == nat.SK_OK, err
    # AoSoA with casts
    t = sk.Collection(wl.TRACK_SCHEMA, ly.AOS)
    t.resize(1000)
    ao = cv.Aosoa.__new__(cv.Aosoa)  # geometry only: no device buffer needed for the check
    ao.n, ao.lanes = 1000, 128
    ao.fields = [cv.AosoaField("pz", "f32"), cv.AosoaField("px", "f32"), cv.AosoaField("charge", "i64")]
    ao.block_off = [0, 512, 1024]
    ao.tile_bytes = 2048

    class _Buf:
        ptr = 1 << 20  # never dereferenced: the check only plans and compiles

    ao.buffer = _Buf()
    st, src, err = _spec_check(cv._aosoa_desc(t.layout, ao, True))
    assert st == nat.SK_OK and "cast_bits(" in src, err
    # per_field <-> AoSoA: the 4-records-per-thread block transform, both directions
    tp = sk.Collection(wl.TRACK_SCHEMA, ly.PER_FIELD)
    tp.resize(1000)
    for to in (True, False):
        st, src, err = _spec_check(cv._aosoa_desc(tp.layout, ao, to))
        assert st == nat.SK_OK and "(r0 >> 7) * 2048" in src and "uint4" in src, err  # T = 128 baked in


# ---- the C-ABI library ---------------------------------------------------------------------

def _header_functions():
    text = open(os.path.join(ROOT, "include", "soakit_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(nat.LIB_PATH)
    names = _header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(nat.exported_names()) == names  # the ctypes binding covers the header exactly


def test_library_loads_and_reports_no_device_cleanly():
    lib = nat.lib()
    assert lib.sk_version() == 0x000100
    n = ctypes.c_int(-1)
    st = lib.sk_device_count(ctypes.byref(n))
    assert st in (nat.SK_OK, nat.SK_ERR_NO_DEVICE, nat.SK_ERR_CUDA)
    if st != nat.SK_OK:
        assert n.value == 0 and lib.sk_last_error()


def test_prepare_refuses_pageable_endpoints():
    """A CUDA graph cannot capture pageable host copies: refused before anything runs."""
    src = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.host())
    src.resize(4)
    dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, mc.ContextInfo.host())
    with pytest.raises(sk.TransferError):
        tr.prepare(dst, src)


def test_move_collection_copies_then_clears_source():
    """move_collection (transfer.py:119-124): copy, then clear the source under engine_ops; storage stays."""
    src = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, mc.ContextInfo.host())
    src.resize(6)
    src.column("seed").np[:] = np.arange(6, dtype=np.uint64) * 7
    want = src.dump()
    dst = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, mc.ContextInfo.host())
    assert tr.move_collection(dst, src) == "bulk-same-kind"
    assert dst.dump() == want
    assert src.size() == 0 and src.capacity() >= 6


def test_skev_event_files_round_trip_with_the_reference(tmp_path):
    """load_events / save_events speak the reference's SKEV format (events.py:147-197) both ways."""
    from skhelp import import_soakit

    soakit = import_soakit()
    if soakit is None:
        pytest.skip("soakit (the reference package) is not installed")
    from soakit.detector import events as ev

    specs = [ev.EventSpec(37, 11, 5, 0.01), ev.EventSpec(37, 11, 6, 0.02)]
    paths = [tmp_path / f"e{i}.skev" for i in range(2)]
    for sp, p in zip(specs, paths):
        ev.save_event(ev.generate_event(sp), p)
    coll = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, mc.ContextInfo.host())
    got = sensor.load_events(paths, coll)
    assert got == [(37, 11, 5, 0.01), (37, 11, 6, 0.02)]
    for i, (sp, p) in enumerate(zip(specs, paths)):
        want = ev.load_event(p)
        sl = slice(i * 407, (i + 1) * 407)
        for name in ("type", "counts", "noisy", "parameter_A", "parameter_B", "noise_A", "noise_B"):
            leaf = name if name in ("type", "counts") else "calibration_data." + name
            assert coll.column(leaf).np[sl].tobytes() == getattr(want, name).tobytes(), name
    assert not coll.column("energy").np.any()
    out = [tmp_path / f"o{i}.skev" for i in range(2)]
    sensor.save_events(coll, out, got)
    for a, b in zip(paths, out):
        assert a.read_bytes() == b.read_bytes()
    bad = tmp_path / "bad.skev"
    bad.write_bytes(paths[0].read_bytes() + b"x")
    with pytest.raises(ValueError):
        sensor.load_events([bad], coll)


def test_return_pool_recycles_and_survives_finalizers_inside_allocation(monkeypatch):
    """memctx.host_return_array's pool on host stand-ins for page-locked memory: buffers come back only when
    every array viewing them is gone, the pool keeps at most keep_bytes, and a garbage-collector finalizer
    that runs while the pool is handing out a buffer cannot deadlock it (finalizers take no lock)."""
    import gc

    live = {}

    def alloc(nbytes):
        buf = (ctypes.c_uint8 * nbytes)()
        ptr = ctypes.addressof(buf)
        live[ptr] = buf
        return ptr

    freed = []
    monkeypatch.setattr(mc.nat, "host_alloc_pinned", alloc)
    monkeypatch.setattr(mc.nat, "host_free_pinned", lambda p: freed.append(live.pop(p) is not None))
    pool = mc._ReturnPool(keep_bytes=8 << 20)
    n = (3 << 20) // 4  # 3 MB of float32 -> the 4 MB size class
    a = pool.array(n, np.float32)
    a[:] = 1.0
    view = a[5:9]
    pa = a.ctypes.data
    del a
    gc.collect()
    b = pool.array(n, np.float32)
    assert b.ctypes.data != pa and view.tolist() == [1.0] * 4  # the view keeps the first buffer out
    del view, b
    gc.collect()
    c = pool.array(n, np.float32)
    assert c.ctypes.data in live  # recycled
    # a cycle whose collection releases a pooled buffer, collected from inside array() (gc.collect runs
    # finalizers synchronously): array() must not deadlock, and the buffer comes back on the next call
    holder = [pool.array(n, np.float32)]
    holder.append(holder)
    del holder
    orig_alloc = mc.nat.host_alloc_pinned

    def alloc_and_collect(nbytes):
        gc.collect()
        return orig_alloc(nbytes)

    monkeypatch.setattr(mc.nat, "host_alloc_pinned", alloc_and_collect)
    d = pool.array(1 << 20, np.uint8)  # a new size class: allocates, which collects the cycle
    assert d.size == 1 << 20
    # beyond keep_bytes returned buffers are freed rather than kept
    many = [pool.array(n, np.float32) for _ in range(4)]
    del many, c, d
    gc.collect()
    pool.array(16, np.uint8)  # below RETURN_POOL_MIN: plain numpy, but drains nothing
    pool.array(n, np.float32)  # drains the returns: 8 MB kept, the rest freed
    assert pool._kept <= 8 << 20 and freed


def _seed_ratio(e, z):
    """the reconstruction tile pass's division-free seed test (sk_reco.cu seed_ratio), restated"""
    t = z.astype(np.float64) * (5.0 + 2.0 ** -22)
    ed = e.astype(np.float64)
    zero = (z == 0) & (e != 0) & ~np.isnan(e) & ((e > 0) != np.signbit(z))
    return np.where(z > 0, ed > t, np.where(z < 0, ed < t, zero))


def test_division_free_seed_test_equals_numpy_f32_division():
    """e / z > 5 in numpy f32 (reconstruct.py:62-66) == the f64 product test, on random values, values one
    ulp either side of the 5 + 2^-22 midpoint, denormals, zeros of both signs, infinities and NaN"""
    rng = np.random.default_rng(5)
    z = rng.standard_normal(2_000_000).astype(np.float32) * np.float32(10) ** rng.integers(-40, 38, 2_000_000)
    z = z.astype(np.float32)
    e = (z.astype(np.float64) * (5.0 + 2.0 ** -22)).astype(np.float32)  # right at the rounding boundary
    e = np.concatenate([e, np.nextafter(e, np.float32(np.inf)), np.nextafter(e, np.float32(-np.inf)),
                        rng.standard_normal(2_000_000).astype(np.float32) * 50])
    z = np.concatenate([z, z, z, z])
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 3.4e38, -3.4e38, 5.0, 1.0],
                        np.float32)
    e = np.concatenate([e, np.repeat(specials, specials.size)])
    z = np.concatenate([z, np.tile(specials, specials.size)])
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        want = (e / z) > np.float32(5)
    assert np.array_equal(_seed_ratio(e, z), want)
