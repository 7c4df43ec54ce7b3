"""The reference package's own API on the B200 (executed).

soakit's copy_collection / move_collection / Collection size operations /
coll.funcs.* are called unmodified after paper_2511_04853_b200.soakit_plugin
registered the cuda + pinned contexts, the b200-convert spec and the
sensor_funcs behaviors. Expected values come from soakit's own CPU path on
the same inputs."""

import itertools

import numpy as np
import pytest

from skhelp import import_soakit

soakit = import_soakit()
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(soakit is None, reason="soakit (the reference package) is not installed")]


@pytest.fixture(scope="module")
def sp():
    from paper_2511_04853_b200 import soakit_plugin

    soakit_plugin.install()
    return soakit_plugin


def _event(w, h, seed, density=0.002):
    from soakit.detector import events

    return events.generate_event(events.EventSpec(w, h, seed, density))


@pytest.mark.parametrize("w,h,seed", [(64, 64, 3), (436, 436, 7)])
def test_prepare_phase_through_soakit_on_cuda(sp, w, h, seed):
    """bench.py:174-178 with ContextInfo.cuda in place of mockdev, plus the AoS -> SoA conversion the
    reference cannot do off-host: pinned AoS -> cuda per_field (b200-convert), calibrate + noise on the
    device, copy back, everything bit-equal to soakit's CPU functions."""
    from soakit.detector import reconstruct as rc
    from soakit.detector import schemas as ds

    C, tr, mc = soakit.Collection, soakit.transfer, soakit.memctx
    ev = _event(w, h, seed)
    ref = C(ds.SENSOR_SCHEMA, "per_field")
    rc.fill_sensor_collection(ref, ev)
    src = C(ds.SENSOR_SCHEMA, "aos", sp.pinned_info())
    assert tr.copy_collection(src, ref) == "b200-convert"
    ds.calibrate_collection(ref)
    want_noise = ds.noise_for_collection(ref)
    dev = C(ds.SENSOR_SCHEMA, "per_field", sp.cuda_info(0))
    assert tr.copy_collection(dev, src) == "b200-convert"
    with mc.execution_scope("cuda"):
        dev.funcs.calibrate_energy()
        noise = dev.funcs.get_noise()
    assert noise.tobytes() == want_noise.tobytes()
    back = C(ds.SENSOR_SCHEMA, "per_field")
    assert tr.copy_collection(back, dev) == "bulk-same-kind"
    assert back.column("energy").read().tobytes() == ref.column("energy").read().tobytes()
    assert back.dump() == ref.dump()
    # object targets on a device record
    rec = w * h // 2 + 3
    with mc.execution_scope("cuda"):
        dev.record(rec).funcs.calibrate_energy()
        one = dev.record(rec).funcs.get_noise()
    assert np.float32(one).tobytes() == want_noise[rec].tobytes()


def _particles(n, seed):
    from soakit.detector import schemas as ds

    rng = np.random.default_rng(seed)
    c = soakit.Collection(ds.PARTICLE_SCHEMA, "aos")
    c.resize(n)
    c.layout._struct_buf._data[: n * 64] = rng.integers(0, 256, n * 64, dtype=np.uint8)
    c.jagged_fill("sensors", [rng.integers(0, 2**63, rng.integers(0, 5), dtype=np.uint64) for _ in range(n)])
    return c


def test_transfer_matrix_through_soakit(sp):
    """C4 (test_acceptance.py:504-552) through soakit's dispatcher with cuda and pinned endpoints: every
    ordered pair of 9 endpoints round-trips dump-identical (AoS destinations off-host included)."""
    from soakit.detector import schemas as ds

    C, tr = soakit.Collection, soakit.transfer
    n = 29
    base = _particles(n, 3)
    want = base.dump()
    total = base.jagged_size("sensors")
    infos = {"host": soakit.memctx.ContextInfo.host(), "pinned": sp.pinned_info(), "cuda": sp.cuda_info(0)}

    def make(kind, ctx):
        arena = soakit.layouts.ArenaSpec({soakit.schema.MAIN_TAG: n + 3, "sensors": total + 5}) if kind == "arena" else None
        return C(ds.PARTICLE_SCHEMA, kind, infos[ctx], arena)

    eps = list(itertools.product(["aos", "per_field", "arena"], infos))
    for (k1, c1), (k2, c2) in itertools.product(eps, eps):
        a, b = make(k1, c1), make(k2, c2)
        tr.copy_collection(a, base)
        tr.copy_collection(b, a)
        h = C(ds.PARTICLE_SCHEMA, "per_field")
        tr.copy_collection(h, b)
        assert h.dump() == want, (k1, c1, k2, c2)


def test_size_ops_and_move_on_cuda_through_soakit(sp):
    """Collection.insert/erase/resize on a cuda-resident soakit collection run through the plugin's
    memset + overlap-safe copiers and match the same ops on a host collection; move_collection clears
    the source (transfer.py:119-124). Sensor records: soakit's own jagged prefix upkeep indexes the
    prefix column from Python (collection.py:444-446), which device memory does not allow -- jagged
    size changes on device data go through this package's Collection instead."""
    from soakit.detector import reconstruct as rc
    from soakit.detector import schemas as ds

    C, tr, mc = soakit.Collection, soakit.transfer, soakit.memctx
    host = C(ds.SENSOR_SCHEMA, "per_field")
    rc.fill_sensor_collection(host, _event(37, 11, 5))
    dev = C(ds.SENSOR_SCHEMA, "per_field", sp.cuda_info(0))
    tr.copy_collection(dev, host)
    ops = [("insert_records", 5, 3), ("erase_records", 10, 7), ("resize", 500), ("erase_records", 0, 4),
           ("insert_records", 300, 150), ("shrink_to_fit",)]
    for op, *args in ops:
        getattr(host, op)(*args)
        with mc.execution_scope("cuda"):
            getattr(dev, op)(*args)
    back = C(ds.SENSOR_SCHEMA, "per_field")
    tr.copy_collection(back, dev)
    assert back.dump() == host.dump()
    moved = C(ds.SENSOR_SCHEMA, "aos", sp.cuda_info(0))
    assert tr.move_collection(moved, dev) == "b200-convert"
    assert dev.size() == 0
    again = C(ds.SENSOR_SCHEMA, "per_field")
    tr.copy_collection(again, moved)
    assert again.dump() == host.dump()
    parts = _particles(33, 4)
    dp = C(ds.PARTICLE_SCHEMA, "per_field", sp.cuda_info(0))
    assert tr.move_collection(dp, parts) == "b200-convert"
    assert parts.size() == 0


def _soakit_schema(rng, k):
    S = soakit.schema
    types = [S.BOOL, S.U8, S.U16, S.U32, S.U64, S.I32, S.I64, S.F32, S.F64, S.enum_type("E", 300)]
    props = []
    for i in range(int(rng.integers(1, 9))):
        kind = rng.random()
        t = types[int(rng.integers(0, len(types)))]
        if kind < 0.6:
            props.append(S.declare_per_item(f"p{i}", t))
        elif kind < 0.8:
            props.append(S.declare_array(f"a{i}", int(rng.integers(1, 5)), t))
        else:
            props.append(S.declare_subgroup(f"g{i}", [S.declare_per_item("u", t),
                                                     S.declare_per_item("v", types[int(rng.integers(0, 9))])]))
    if rng.random() < 0.4:
        props.append(S.declare_jagged("jv", S.I32, types[int(rng.integers(1, 9))]))
    if rng.random() < 0.3:
        props.append(S.declare_global("gl", types[int(rng.integers(1, 9))]))
    return S.Schema(f"R{k}", tuple(props))


def _planes(coll):
    """every plane's live bytes, leaf#slot -> bytes (host-visible per_field collection)"""
    lay = coll.layout
    out = {}
    for lf in coll.plan.leaves:
        n = lay.plane_len(lf) * lf.value_type.size_bytes
        for k in range(lay.plane_count(lf)):
            buf, off = lay._plane_region(lf, k)
            out[f"{lf.dotted}#{k}"] = bytes(buf._data[off:off + n])
    return out


@pytest.mark.parametrize("k", range(16))
def test_random_schemas_match_soakit_cpu_path(sp, k):
    """Random plans (mixed scalar types, fixed arrays, sub-groups, a jagged vector, a global, odd packed
    strides), random records: soakit's own CPU conversion (per-leaf-default, host AoS -> host per_field) is
    the expected result; the B200 path through soakit's dispatcher is host AoS -> cuda per_field
    (b200-convert) -> cuda AoS (K2, which the reference cannot do off-host) -> cuda per_field -> host. Every
    plane is byte-identical, and the device AoS image equals the input records."""
    C, tr = soakit.Collection, soakit.transfer
    rng = np.random.default_rng(500 + k)
    schema = _soakit_schema(rng, k)
    n = int(rng.integers(1, 2500))
    src = C(schema, "aos")
    src.resize(n)
    stride = src.layout.record_stride
    raw = rng.integers(0, 256, n * stride, dtype=np.uint8)
    src.layout._struct_buf._data[: n * stride] = raw
    if any(t.id == "jv" for t in src.plan.jagged_tags()):
        dt = src.plan.leaf("jv.value").value_type.np_dtype
        src.jagged_fill("jv", [np.frombuffer(rng.integers(0, 256, int(rng.integers(0, 4)) * dt.itemsize,
                                                            dtype=np.uint8).tobytes(), dt) for _ in range(n)])
    if src.plan.has_leaf("gl"):
        src.set_global("gl", 3)
    want = C(schema, "per_field")
    assert tr.copy_collection(want, src) == "per-leaf-default"
    dev = C(schema, "per_field", sp.cuda_info(0))
    assert tr.copy_collection(dev, src) == "b200-convert"
    dev_aos = C(schema, "aos", sp.cuda_info(0))
    assert tr.copy_collection(dev_aos, dev) == "b200-convert"
    dev2 = C(schema, "per_field", sp.cuda_info(0))
    assert tr.copy_collection(dev2, dev_aos) == "b200-convert"
    got = C(schema, "per_field")
    assert tr.copy_collection(got, dev2) == "bulk-same-kind"
    assert _planes(got) == _planes(want), k
    assert got.dump() == want.dump()
    back = C(schema, "aos")
    tr.copy_collection(back, dev_aos)  # cuda AoS -> host AoS: bulk-same-kind
    assert bytes(back.layout._struct_buf._data[: n * stride]) == raw.tobytes()
