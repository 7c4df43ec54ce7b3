"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the dev container, where the reference package is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every array saved here is produced by soakit 0.1.0 itself (/root/reference/pkg/src)
through its public path: copy_collection (per-leaf-default), jagged_fill,
import_external, calibrate_collection / noise_for_collection under
execution_scope("mockdev"), generate_event / mix_stream, and the layout
geometry. The fixtures travel with the repo; the GPU box never reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import soakit as sk  # noqa: E402
from soakit import detector as det  # noqa: E402
from soakit import layouts as ly  # noqa: E402
from soakit import memctx as mc  # noqa: E402
from soakit import schema as sc  # noqa: E402
from soakit import transfer as tr  # noqa: E402


def save(name: str, **arrays) -> None:
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def leaf_planes(coll) -> dict[str, np.ndarray]:
    """Raw bytes of every plane [0, plane_len) of every leaf of a per_field collection."""
    lay = coll._layout
    out = {}
    for leaf in coll.plan.leaves:
        for k in range(lay.plane_count(leaf)):
            out[f"{leaf.dotted}#{k}"] = np.array(lay._plane_view(leaf, k)).view(np.uint8).copy()
    return out


def obj8() -> None:
    schema = sc.Schema("Obj8", tuple(sc.declare_per_item(f"f{i}", sc.F32 if i % 2 == 0 else sc.I32) for i in range(8)))
    n = 4099  # not a multiple of any tile size: exercises the tail
    rng = np.random.default_rng(1234)
    raw = rng.integers(0, 256, n * 32, dtype=np.uint8)
    # sprinkle float specials into the f32 fields
    words = raw.view(np.uint32).reshape(n, 8)
    specials = np.array([0, 0x80000000, 0x7F800000, 0xFF800000, 1, 0x807FFFFF, 0x7FC00001, 0x7F800ABC], np.uint32)
    for f in (0, 2, 4, 6):
        hit = rng.random(n) < 0.05
        words[hit, f] = specials[rng.integers(0, specials.size, int(hit.sum()))]
    src = sk.Collection(schema, ly.AOS)
    src.resize(n)
    src._layout._struct_buf._data[: n * 32] = raw
    dst = sk.Collection(schema, ly.PER_FIELD)
    name = tr.copy_collection(dst, src)
    assert name == "per-leaf-default", name
    planes = leaf_planes(dst)
    # reverse direction: planes -> aos
    back = sk.Collection(schema, ly.AOS)
    assert tr.copy_collection(back, dst) == "per-leaf-default"
    aos_back = np.array(back._layout._struct_buf._data[: n * 32])
    assert aos_back.tobytes() == raw.tobytes()
    save("obj8.npz", aos=raw, **{f"plane:{k}": v for k, v in planes.items()}, n=np.int64(n))


def particle() -> None:
    schema = det.PARTICLE_SCHEMA
    n = 1000
    rng = np.random.default_rng(99)
    src = sk.Collection(schema, ly.AOS)
    src.resize(n)
    stride = src._layout.record_stride
    raw = rng.integers(0, 256, n * stride, dtype=np.uint8)
    src._layout._struct_buf._data[: n * stride] = raw
    segs = [rng.integers(0, 2**63, rng.integers(0, 9), dtype=np.uint64) for _ in range(n)]
    src.jagged_fill("sensors", segs)
    dst = sk.Collection(schema, ly.PER_FIELD)
    assert tr.copy_collection(dst, src) == "per-leaf-default"
    planes = leaf_planes(dst)
    arena = sk.Collection(schema, ly.ARENA, None, ly.ArenaSpec({sc.MAIN_TAG: n + 7, "sensors": 6000}, 64))
    assert tr.copy_collection(arena, src) == "per-leaf-default"
    save("particle.npz", aos=raw, stride=np.int64(stride), n=np.int64(n),
         pool_total=np.int64(src.jagged_size("sensors")),
         **{f"plane:{k}": v for k, v in planes.items()},
         arena_image=np.array(arena._layout._buf._data))


def geometry() -> None:
    out = {}
    plan = det.PARTICLE_PLAN
    for align in (16, 64, 4096):
        spec = ly.ArenaSpec({sc.MAIN_TAG: 10, "sensors": 33}, align)
        lay = ly.build_layout(ly.ARENA, plan, None, spec)
        out[f"arena_offsets_{align}"] = np.array([lay.leaf_offset(lf) for lf in plan.leaves], np.int64)
        out[f"arena_total_{align}"] = np.int64(lay.total_bytes)
        lay.free()
    lay = ly.build_layout(ly.AOS, plan)
    out["particle_stride"] = np.int64(lay.record_stride)
    lay.free()
    lay = ly.build_layout(ly.AOS, det.SENSOR_PLAN)
    out["sensor_stride"] = np.int64(lay.record_stride)
    lay.free()
    lay = ly.build_layout(ly.PER_FIELD, plan)
    caps = []
    for n in (1, 5, 17):
        lay.resize(sc.MAIN_TAG, n)
        caps.append(lay.capacity(sc.MAIN_TAG))
    out["growth"] = np.array(caps, np.int64)
    lay.free()
    out["particle_leaves"] = np.array([f"{lf.dotted}|{lf.value_type.np_dtype.str}|{lf.size_tag}|"
                                       f"{lf.extent_multiplier}|{lf.role}" for lf in plan.leaves])
    out["sensor_leaves"] = np.array([f"{lf.dotted}|{lf.value_type.np_dtype.str}|{lf.size_tag}|"
                                     f"{lf.extent_multiplier}|{lf.role}" for lf in det.SENSOR_PLAN.leaves])
    save("geometry.npz", **out)


def sensors() -> None:
    for (w, h, seed, dens) in ((16, 16, 5, 0.01), (64, 64, 3, 0.002), (101, 37, 11, 0.004)):
        ev = det.generate_event(det.EventSpec(w, h, seed=seed, particle_density=dens))
        aos = det.HandwrittenAosPipeline()
        aos.fill(ev)
        aos_bytes = np.frombuffer(aos.sensors.tobytes(), np.uint8).copy()  # energy still 0 (baselines.py:140)
        host = sk.Collection(det.SENSOR_SCHEMA, ly.AOS)
        det.fill_sensor_collection(host, ev)
        assert np.array(host._layout._struct_buf._data[: w * h * 30]).tobytes() == aos.sensors.tobytes()
        dev = sk.Collection(det.SENSOR_SCHEMA, ly.PER_FIELD, mc.ContextInfo.mockdev())
        assert tr.copy_collection(dev, host) == "per-leaf-default"
        with mc.execution_scope(mc.MOCKDEV):
            dev.funcs.calibrate_energy()
            noise = dev.funcs.get_noise()
            energy = np.array(dev.column("energy").read())
        aos.calibrate()
        assert energy.tobytes() == np.ascontiguousarray(aos.sensors["energy"]).tobytes()
        assert noise.tobytes() == aos.noise().tobytes()
        cols = {k: getattr(ev, k) for k in ("type", "counts", "noisy", "parameter_A", "parameter_B", "noise_A",
                                              "noise_B")}
        save(f"sensor_{w}x{h}_s{seed}.npz", aos=aos_bytes,
             energy=energy, noise=noise, w=np.int64(w), h=np.int64(h), seed=np.int64(seed),
             density=np.float64(dens), **{f"ev:{k}": v for k, v in cols.items()})


def jagged() -> None:
    rng = np.random.default_rng(7)
    out = {}
    for label, itype, n in (("i32", sc.I32, 3000), ("u8", sc.U8, 100), ("u16", sc.U16, 1500), ("i64", sc.I64, 50)):
        schema = sc.Schema("J", (sc.declare_per_item("seed", sc.U64), sc.declare_jagged("members", itype, sc.U64)))
        c = sk.Collection(schema, ly.PER_FIELD)
        c.resize(n)
        lens = rng.integers(0, 21, n)
        lens[rng.random(n) < 0.05] = 0
        segs = [rng.integers(0, 2**64 - 1, l, dtype=np.uint64) for l in lens]
        c.jagged_fill("members", segs)
        out[f"{label}:lens"] = lens.astype(np.int32)
        out[f"{label}:pool_in"] = np.concatenate(segs) if segs else np.empty(0, np.uint64)
        out[f"{label}:prefix"] = c.prefix_sums("members")
        out[f"{label}:pool"] = np.array(c.column("members").read())
    # multi-leaf members through import_external (transfer.py:297-320)
    schema = sc.Schema("Cluster2", (sc.declare_per_item("seed", sc.U64),
                                    sc.declare_jagged("hits", sc.I32, [sc.declare_per_item("adc", sc.I32),
                                                                        sc.declare_per_item("t", sc.F32)])))
    n = 500
    recs = []
    for i in range(n):
        m = int(rng.integers(0, 12))
        recs.append({"seed": i, "adc": rng.integers(-2**31, 2**31, m).tolist(),
                     "t": rng.standard_normal(m).astype(np.float32).tolist()})
    binding = tr.ExternalBinding(extractors={"seed": lambda r: r["seed"], "hits.adc": lambda r: r["adc"],
                                             "hits.t": lambda r: r["t"]})
    c = sk.Collection(schema, ly.PER_FIELD)
    tr.import_external(c, binding, recs)
    out["hits:lens"] = np.array([len(r["adc"]) for r in recs], np.int32)
    out["hits:adc_in"] = np.array([v for r in recs for v in r["adc"]], np.int32)
    out["hits:t_in"] = np.array([v for r in recs for v in r["t"]], np.float32)
    out["hits:prefix"] = c.prefix_sums("hits")
    out["hits:adc"] = np.array(c.column("hits.adc").read())
    out["hits:t"] = np.array(c.column("hits.t").read())
    save("jagged.npz", **out)


def particles() -> None:
    """reconstruct_arrays (detector/reconstruct.py:53-136) on calibrated events,
    including a dense event where deposit windows overlap heavily."""
    for (w, h, seed, dens) in ((16, 16, 5, 0.01), (64, 64, 3, 0.002), (101, 37, 11, 0.004), (160, 120, 21, 0.02)):
        ev = det.generate_event(det.EventSpec(w, h, seed=seed, particle_density=dens))
        aos = det.HandwrittenAosPipeline()
        aos.fill(ev)
        aos.calibrate()
        s = aos.sensors
        p = det.reconstruct_arrays(s["energy"], aos.noise(), s["type"], s["calibration_data"]["noisy"], w, h)
        save(f"particles_{w}x{h}_s{seed}.npz", w=np.int64(w), h=np.int64(h), seed=np.int64(seed),
             density=np.float64(dens), energy=p.energy, x=p.x, y=p.y, origin=p.origin, x_variance=p.x_variance,
             y_variance=p.y_variance, significance=p.significance, E_contribution=p.E_contribution,
             noisy_count=p.noisy_count, sensor_lens=np.array([a.size for a in p.sensors], np.int32),
             sensors=np.concatenate(p.sensors) if len(p.sensors) else np.empty(0, np.uint64))


def splitmix() -> None:
    out = {}
    for seed in (0, 1, 0xDEADBEEF, (1 << 64) - 1):
        out[f"seed{seed}"] = det.events.mix_stream(seed, 0, 64)
        out[f"seed{seed}_off17"] = det.events.mix_stream(seed, 17, 10)
    save("splitmix.npz", **out)


if __name__ == "__main__":
    obj8()
    particle()
    geometry()
    sensors()
    jagged()
    particles()
    splitmix()
