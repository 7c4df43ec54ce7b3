"""The paper's case study on the B200: sensor/particle schemas, the per-object
calibration/noise kernel (K5) and the fused transfer + calibrate path.

Schemas follow detector/schemas.py:56-90 (Listings 1, 2, 4 of the paper);
SENSOR_AOS_DTYPE is the 30-byte packed record of detector/baselines.py:19-35,
byte-identical to AosLayout's image of the Sensor plan.

The collection-target behaviors registered under "sensor_funcs" launch K5 on
CUDA-resident collections. Host-resident collections are refused with
AccessError: in this framework the case-study kernel is device code, as
inside the reference's execution_scope(mockdev) (memctx.py:369-395).
"""

from __future__ import annotations

import ctypes as C
import math
import struct

import numpy as np

from . import _native as nat
from . import behaviors as bh
from . import convert as cv
from . import layouts as ly
from . import memctx
from . import schema as sc
from .devarray import DeviceArray
from .errors import AccessError, UnsupportedTransferError

NUM_SENSOR_TYPES = 4
SENSOR_TYPE = sc.enum_type("SensorType", NUM_SENSOR_TYPES)

SENSOR_AOS_DTYPE = np.dtype([
    ("type", "u1"), ("counts", "<u8"), ("energy", "<f4"),
    ("calibration_data", [("noisy", "?"), ("parameter_A", "<f4"), ("parameter_B", "<f4"),
                          ("noise_A", "<f4"), ("noise_B", "<f4")]),
])

_COUNTS, _ENERGY, _NOISY = "counts", "energy", "calibration_data.noisy"
_A, _B = "calibration_data.parameter_A", "calibration_data.parameter_B"
_NA, _NB = "calibration_data.noise_A", "calibration_data.noise_B"


def _device_planes(coll) -> tuple[int, dict]:
    lay = coll.layout
    if lay.host_visible:
        raise AccessError(
            f"the case-study kernel runs on the B200; move the collection to ContextInfo.cuda() first "
            f"(it is {coll.info.context!r}-resident)"
        )
    if isinstance(lay, ly.AosLayout):
        raise UnsupportedTransferError("case-study kernel reads per_field/arena planes; convert the AoS collection first")
    names = (_COUNTS, _ENERGY, _NOISY, _A, _B, _NA, _NB)
    if coll.plan is SENSOR_PLAN or coll.plan == SENSOR_PLAN:  # the usual case: one batched address pass
        return lay.device, dict(zip(names, lay.main_slot_addresses(_SENSOR_SLOTS)))
    return lay.device, {k: lay.plane_address(coll.plan.leaf(k), 0) for k in names}


def calibrate_collection(coll, sync: bool = True) -> None:
    """energy = A * f32(counts) + B on the device (detector/schemas.py:29-33)."""
    dev, p = _device_planes(coll)
    n = coll.size()
    nat.call("sk_sensor_calibrate", n, p[_COUNTS], p[_A], p[_B], p[_ENERGY], nat.stream(dev))
    if sync:
        nat.sync(dev)


def noise_for_collection(coll, out: DeviceArray | None = None, sync: bool = True) -> DeviceArray:
    """Per-sensor noise as a device f32 array (detector/schemas.py:36-41)."""
    dev, p = _device_planes(coll)
    n = coll.size()
    if out is None:
        out = DeviceArray(n, np.float32, memctx.ContextInfo.cuda(dev))
    nat.call("sk_sensor_noise", n, p[_ENERGY], p[_NA], p[_NB], p[_NOISY], out.ptr, nat.stream(dev))
    if sync:
        nat.sync(dev)
    return out


def transfer_calibrate(dst, src, noise: DeviceArray | None = None, sync: bool = True) -> DeviceArray:
    """Fused K1+K5: AoS sensor records (any placement) -> per_field/arena planes
    on the device with energy calibrated, plus the noise column, one HBM pass.

    Equivalent to copy_collection(dst, src) followed by calibrate_energy() and
    get_noise() (bench.py:174-178 prepare phase)."""
    sl, dl = src.layout, dst.layout
    if not isinstance(sl, ly.AosLayout) or isinstance(dl, ly.AosLayout):
        raise UnsupportedTransferError("fused sensor path converts AoS records into planes")
    if dl.host_visible:
        raise AccessError("fused sensor path writes a device-resident destination")
    if dst.plan != src.plan or dst.plan != SENSOR_PLAN:
        raise UnsupportedTransferError("fused sensor path needs the Sensor plan on both sides")
    from .transfer import _cached_desc, _match_sizes  # same reserve-then-size contract as copy_collection

    _match_sizes(dst, src)
    n = sl.size(sc.MAIN_TAG)
    dev = dl.device
    if noise is None:
        noise = DeviceArray(n, np.float32, memctx.ContextInfo.cuda(dev))
    desc = _cached_desc(dl, sl, n)
    idx = _FUSED_FIELDS
    if n:
        nat.call("sk_sensor_convert_calibrate", C.byref(desc), *idx, noise.ptr, dev, nat.stream(dev))
    dst._bump()
    if sync:
        nat.sync(dev)
    return noise


def footprint() -> list[float]:
    """The reference's 5x5 deposit footprint, evaluated with the same libm
    (events.py:31-33), row-major."""
    return [math.exp(-(dx * dx + dy * dy) / 2.88) for dy in range(-2, 3) for dx in range(-2, 3)]


def generate_events(coll, width: int, height: int, seeds, density: float = 0.0, sync: bool = True) -> None:
    """Fill a device-resident Sensor collection with len(seeds) events of
    width x height cells generated on the GPU, event-major, energy zeroed:
    byte-identical to generate_event + fill_sensor_collection
    (detector/events.py:85-133, detector/reconstruct.py:142-154) per event."""
    dev, p = _device_planes(coll)
    seeds = [int(s) for s in seeds]
    n = width * height
    total = n * len(seeds)
    lay = coll.layout
    with lay.engine_ops():
        lay.reserve(sc.MAIN_TAG, total)
        lay._set_sizes_for_engine({sc.MAIN_TAG: total})
    dev, p = _device_planes(coll)  # reserve may have reallocated the planes
    n_dep = int(round(density * n))
    c_seeds = (C.c_uint64 * max(len(seeds), 1))(*seeds)
    foot = (C.c_double * 25)(*footprint())
    ptype = lay.plane_address(coll.plan.leaf("type"), 0)
    nat.call("sk_sensor_generate", width, height, c_seeds, len(seeds), n_dep, foot, ptype, p[_COUNTS], p[_NOISY],
             p[_A], p[_B], p[_NA], p[_NB], p[_ENERGY], nat.stream(dev))
    coll._bump()
    if sync:
        nat.sync(dev)


def reconstruct_from_collection(sensors, width: int, height: int, out=None, events: int = 1, noise=None):
    """Particle reconstruction on the GPU (detector/reconstruct.py:172-194 /
    reconstruct_arrays 53-136) for `events` calibrated events stored event-major
    in a device-resident Sensor collection. Returns a device per_field Particle
    collection (or fills `out`) with the reference's particles in the
    reference's order, events concatenated; out.event_counts holds the
    per-event particle counts."""
    from .collection import Collection

    dev, p = _device_planes(sensors)
    n = width * height
    if sensors.size() != n * events:
        raise UnsupportedTransferError(f"collection holds {sensors.size()} cells, expected {events} x {n}")
    if noise is None:
        noise = noise_for_collection(sensors, sync=False)
    ptype = sensors.layout.plane_address(sensors.plan.leaf("type"), 0)
    if out is None:
        out = Collection(PARTICLE_SCHEMA, ly.PER_FIELD, memctx.ContextInfo.cuda(dev))
    lay = out.layout
    # the output is written before the host learns the particle count: give it room for a typical run
    # (benchmark events: ~0.27% of the cells become particles, ~20 sensors each), or what it already has
    with lay.engine_ops():
        out.clear()
        lay.reserve(sc.MAIN_TAG, max(1024, n * events // 200))
        lay.reserve("sensors", 24 * lay.capacity(sc.MAIN_TAG))
    handle = C.c_void_p(0)
    m, ncon, rounds, written = C.c_int64(0), C.c_int64(0), C.c_int(0), C.c_int(0)
    nat.call("sk_reco_run", width, height, events, p[_ENERGY], noise.ptr, ptype, p[_NOISY],
             C.byref(_reco_out(out)), dev, nat.stream(dev), C.byref(handle), C.byref(m), C.byref(ncon),
             C.byref(rounds), C.byref(written))
    try:
        m, ncon = m.value, ncon.value
        if not written.value:  # more particles than room: grow the output, write again
            with lay.engine_ops():
                lay.reserve(sc.MAIN_TAG, m)
                lay.reserve("sensors", ncon)
            nat.call("sk_reco_write", handle, C.byref(_reco_out(out)), nat.stream(dev))
        with lay.engine_ops():
            lay._set_sizes_for_engine({sc.MAIN_TAG: m, "sensors": ncon})
        out._bump()
        counts = (C.c_int64 * max(events, 1))()
        nat.call("sk_reco_event_counts", handle, counts)
        out.event_counts = list(counts)[:events]
        out.reco_rounds = rounds.value
    finally:
        nat.call("sk_reco_free", handle, nat.stream(dev))
    if not written.value:
        nat.sync(dev)
    return out


def _reco_out(coll) -> "nat.RecoOut":
    """The sk_reco_out view of a device per_field Particle collection, at its current capacities."""
    lay = coll.layout
    addr = lambda leaf, k=0: lay.plane_address(PARTICLE_PLAN.leaf(leaf), k)  # noqa: E731
    o = nat.RecoOut()
    o.energy, o.x, o.y, o.origin = addr("energy"), addr("x"), addr("y"), addr("origin")
    o.x_variance, o.y_variance = addr("x_variance"), addr("y_variance")
    for k in range(4):
        o.significance[k] = addr("significance.value", k)
        o.e_contribution[k] = addr("E_contribution.value", k)
        o.noisy_count[k] = addr("noisy_count.value", k)
    pleaf = PARTICLE_PLAN.leaf("sensors.prefix_sum")
    o.sensor_prefix = lay.plane_address(pleaf, 0)
    o.sensor_prefix_type = nat.TYPE_CODES[pleaf.value_type.storage_code]
    o.sensor_pool = addr("sensors.value")
    o.particle_capacity = lay.capacity(sc.MAIN_TAG)
    o.pool_capacity = lay.capacity("sensors")
    return o


def fused_transfer(dst, src, opts=None) -> None:
    """copy_collection(dst, src, {"fuse": "sensor_funcs"}): the AoS -> planes
    conversion computes the calibrated energy and the noise in the same HBM
    pass (K1+K5, transfer_calibrate). dst remembers the noise column for the
    current content, so the reference's prepare sequence -- copy_collection,
    funcs.calibrate_energy(), funcs.get_noise() (bench.py:174-178) -- costs
    one pass: calibrate_energy() finds the energy already calibrated and
    get_noise() returns the column (the same device array until dst's next
    transfer; free() it and the next fused transfer allocates another). Any
    change to dst (a size change, a transfer, a write through the API) bumps
    its epoch and drops the markers."""
    noise = getattr(dst, "_fused_noise", (None, None))[1]
    if noise is None or not noise.buffer.live or noise.n != src.size():
        if noise is not None:
            noise.free()
        noise = None
    noise = transfer_calibrate(dst, src, noise, sync=not (opts or {}).get("async"))
    dst._fused_noise = (dst._epoch + 1, noise)  # copy_collection bumps the epoch once more after us
    dst._fused_calibrated = dst._epoch + 1


def _fresh(coll, attr: str) -> bool:
    mark = getattr(coll, attr, None)
    stamp = mark[0] if isinstance(mark, tuple) else mark
    return stamp is not None and stamp == coll._epoch


def _calibrate_behavior(coll) -> None:
    if _fresh(coll, "_fused_calibrated"):
        return  # energy is a pure function of counts, A and B: the fused pass already wrote it
    calibrate_collection(coll)


def _noise_behavior(coll) -> DeviceArray:
    if _fresh(coll, "_fused_noise") and coll._fused_noise[1].buffer.live:
        return coll._fused_noise[1]
    return noise_for_collection(coll)


def _one_record(view) -> tuple[int, dict, int]:
    """(device, plane addresses, record index) of a record view on a device collection."""
    coll = view._coll
    dev, planes = _device_planes(coll)
    return dev, planes, view.index


def _calibrate_object(view) -> None:
    """Per-object form (detector/schemas.py:15-17). Host records: numpy scalar
    arithmetic as in the reference; device records: K5 over that one record."""
    if view._coll.layout.host_visible:
        cal = view.calibration_data
        view.energy = np.float32(cal.parameter_A) * np.float32(view.counts) + np.float32(cal.parameter_B)
        return
    dev, p, i = _one_record(view)
    nat.call("sk_sensor_calibrate", 1, p[_COUNTS] + 8 * i, p[_A] + 4 * i, p[_B] + 4 * i, p[_ENERGY] + 4 * i,
             nat.stream(dev))
    nat.sync(dev)


def _noise_object(view) -> np.float32:
    """Per-object form (detector/schemas.py:20-26)."""
    if view._coll.layout.host_visible:
        cal = view.calibration_data
        e = np.maximum(np.float32(view.energy), np.float32(0.0))
        n = np.float32(cal.noise_A) * np.sqrt(e) + np.float32(cal.noise_B)
        return n * np.float32(2.0) if cal.noisy else n
    dev, p, i = _one_record(view)
    out = DeviceArray(1, np.float32, memctx.ContextInfo.cuda(dev))
    nat.call("sk_sensor_noise", 1, p[_ENERGY] + 4 * i, p[_NA] + 4 * i, p[_NB] + 4 * i, p[_NOISY] + i, out.ptr,
             nat.stream(dev))
    val = out.numpy()[0]
    out.free()
    return val


if not bh.is_registered("sensor_funcs"):
    bh.register_bundle("sensor_funcs", [
        bh.BehaviorFunction("calibrate_energy", bh.TARGET_OBJECT, _calibrate_object),
        bh.BehaviorFunction("calibrate_energy", bh.TARGET_COLLECTION, _calibrate_behavior),
        bh.BehaviorFunction("get_noise", bh.TARGET_OBJECT, _noise_object),
        bh.BehaviorFunction("get_noise", bh.TARGET_COLLECTION, _noise_behavior),
    ])

PARTICLE_AOS_DTYPE = np.dtype([
    ("energy", "<f4"), ("x", "<f4"), ("y", "<f4"), ("origin", "<u8"), ("x_variance", "<f4"),
    ("y_variance", "<f4"), ("significance", "<f4", (4,)), ("E_contribution", "<f4", (4,)), ("noisy_count", "u1", (4,)),
])


def export_particles_from_collection(coll, stage=None) -> tuple[np.ndarray, list]:
    """The external AoS form of a particle collection (detector/baselines.py:104-120):
    the packed particle records (PARTICLE_AOS_DTYPE, baselines.py:37-49) and one
    sensor-index array per particle. A device-resident collection is converted
    to packed records on the B200 (K2) and comes back in one copy per buffer;
    `stage` (a pinned AoS Particle collection) is reused across calls when given."""
    from .collection import Collection
    from .transfer import copy_collection

    if stage is None:
        stage = Collection(PARTICLE_SCHEMA, ly.AOS, memctx.ContextInfo.pinned())
    copy_collection(stage, coll)
    n = stage.size()
    lay = stage.layout
    # plain byte copies into recycled page-locked arrays, then the record view (copying through the
    # structured dtype is 7x slower, fresh pageable arrays fault in every page)
    nrec = n * PARTICLE_AOS_DTYPE.itemsize
    recs = memctx.host_return_array(nrec, np.uint8)
    recs[:] = lay._struct_buf._data[:nrec]
    recs = recs.view(PARTICLE_AOS_DTYPE)
    src_pool = lay._plane_view(stage.plan.leaf("sensors.value"), 0)
    pool = memctx.host_return_array(src_pool.size, src_pool.dtype)
    pool[:] = src_pool
    b = np.array(lay._plane_view(stage.plan.leaf("sensors.prefix_sum"), 0)).astype(np.int64)
    try:  # one view of the pool per particle, made in C (csrc/segpack.cpp)
        from . import _segpack
        return recs, _segpack.split_views(pool, b[: n + 1])
    except ImportError:  # pragma: no cover - not built
        bl = b.tolist()
        return recs, [pool[bl[i]:bl[i + 1]] for i in range(n)]


_EVENT_COLUMNS = ("type", "counts", "noisy", "parameter_A", "parameter_B", "noise_A", "noise_B")

# SKEV event files (detector/events.py:27-29, 147-197): a 32-byte header, then the seven input columns
# one after another -- already the per_field image, so loading is one copy per column
_SKEV_MAGIC, _SKEV_VERSION = b"SKEV", 1
_SKEV_HEADER = struct.Struct("<4sHHIIQd")
_SKEV_DTYPES = (np.dtype("u1"), np.dtype("<u8"), np.dtype("u1"), np.dtype("<f4"), np.dtype("<f4"),
                np.dtype("<f4"), np.dtype("<f4"))


def _leaf_of(name: str) -> str:
    return name if name in ("type", "counts") else "calibration_data." + name


def load_events(paths, coll) -> list[tuple[int, int, int, float]]:
    """Read SKEV event files into a Sensor collection, event-major, energy
    zeroed (the reference's load_event + fill_sensor_collection per event,
    events.py:165-197, reconstruct.py:142-154). Every file must hold the same
    grid. The columns go straight into the planes: a host copy for host
    collections, one host-to-device copy per column for device collections
    (call it from execution_scope("cuda") for those). Returns each file's
    (width, height, seed, density). Errors follow the reference: ValueError for
    a truncated file, a wrong magic or version, or trailing bytes."""
    from .collection import _write_plane

    paths = [str(p) for p in paths]
    raws, specs = [], []
    for path in paths:
        raw = np.fromfile(path, dtype=np.uint8)
        if raw.size < _SKEV_HEADER.size:
            raise ValueError(f"{path}: truncated event file")
        magic, version, _, w, h, seed, density = _SKEV_HEADER.unpack_from(raw.tobytes()[: _SKEV_HEADER.size])
        if magic != _SKEV_MAGIC:
            raise ValueError(f"{path}: not an event file")
        if version != _SKEV_VERSION:
            raise ValueError(f"{path}: unsupported event file version {version}")
        n = w * h
        end = _SKEV_HEADER.size + n * sum(dt.itemsize for dt in _SKEV_DTYPES)
        if end > raw.size:
            raise ValueError(f"{path}: truncated event file")
        if end != raw.size:
            raise ValueError(f"{path}: trailing bytes after event data")
        if specs and (w, h) != specs[0][:2]:
            raise ValueError(f"{path}: grid {w}x{h} differs from {specs[0][0]}x{specs[0][1]}")
        raws.append(raw)
        specs.append((w, h, seed, density))
    n = specs[0][0] * specs[0][1] if specs else 0
    total = n * len(paths)
    if coll.size() != total:
        coll.clear()
        coll.resize(total)
    lay = coll.layout
    lay.check_writable()
    for e, raw in enumerate(raws):
        off = _SKEV_HEADER.size
        for name, dt in zip(_EVENT_COLUMNS, _SKEV_DTYPES):
            col = raw[off : off + n * dt.itemsize].view(dt)
            off += n * dt.itemsize
            _write_plane(lay, coll.plan.leaf(_leaf_of(name)), 0, e * n, col)
        _write_plane(lay, coll.plan.leaf("energy"), 0, e * n, np.zeros(n, np.float32))
    coll._bump()
    return specs


def save_events(coll, paths, specs) -> None:
    """Write each event of a Sensor collection (event-major, grids given by
    specs = [(width, height, seed, density)]) as a SKEV file (events.py:147-162)."""
    from .collection import _read_plane

    lay = coll.layout
    lay.check_readable()
    first = 0
    for path, (w, h, seed, density) in zip(paths, specs):
        n = w * h
        with open(path, "wb") as f:
            f.write(_SKEV_HEADER.pack(_SKEV_MAGIC, _SKEV_VERSION, 0, w, h, seed, density))
            for name, dt in zip(_EVENT_COLUMNS, _SKEV_DTYPES):
                col = _read_plane(lay, coll.plan.leaf(_leaf_of(name)), 0, first, first + n)
                f.write(np.ascontiguousarray(col).astype(dt).tobytes())
        first += n


def fill_sensor_collection(coll, event) -> None:
    """Load one event into a Sensor collection, reusing its size when it
    matches (detector/reconstruct.py:142-154). `event` is the reference's
    EventData (or any object/mapping with its seven columns). Host
    collections are written through their columns as in the reference;
    device collections take one host-to-device copy per plane (call it from
    execution_scope("cuda"), like any device-side size change)."""
    from .collection import _write_plane

    get = (lambda k: event[k]) if isinstance(event, dict) else (lambda k: getattr(event, k))
    spec = event.get("spec") if isinstance(event, dict) else getattr(event, "spec", None)
    n = spec.n_sensors if spec is not None else len(get("type"))
    if coll.size() != n:
        coll.clear()
        coll.resize(n)
    lay = coll.layout
    for name in _EVENT_COLUMNS:
        leaf_path = name if name in ("type", "counts") else "calibration_data." + name
        values = np.asarray(get(name))
        if lay.host_visible:
            coll.column(leaf_path).np[:] = values
        else:
            lay.check_writable()
            _write_plane(lay, coll.plan.leaf(leaf_path), 0, 0, values)
    coll._bump()

SENSOR_SCHEMA = sc.Schema("Sensor", (
    sc.declare_per_item("type", SENSOR_TYPE),
    sc.declare_per_item("counts", sc.U64),
    sc.declare_per_item("energy", sc.F32),
    sc.declare_subgroup("calibration_data", [
        sc.declare_per_item("noisy", sc.BOOL),
        sc.declare_per_item("parameter_A", sc.F32),
        sc.declare_per_item("parameter_B", sc.F32),
        sc.declare_per_item("noise_A", sc.F32),
        sc.declare_per_item("noise_B", sc.F32),
    ]),
    sc.declare_behavior("funcs", "sensor_funcs"),
))

PARTICLE_SCHEMA = sc.Schema("Particle", (
    sc.declare_per_item("energy", sc.F32),
    sc.declare_per_item("x", sc.F32),
    sc.declare_per_item("y", sc.F32),
    sc.declare_per_item("origin", sc.U64),
    sc.declare_jagged("sensors", sc.I32, sc.U64),
    sc.declare_per_item("x_variance", sc.F32),
    sc.declare_per_item("y_variance", sc.F32),
    sc.declare_array("significance", NUM_SENSOR_TYPES, sc.F32),
    sc.declare_array("E_contribution", NUM_SENSOR_TYPES, sc.F32),
    sc.declare_array("noisy_count", NUM_SENSOR_TYPES, sc.U8),
))

SENSOR_PLAN = sc.flatten(SENSOR_SCHEMA)
PARTICLE_PLAN = sc.flatten(PARTICLE_SCHEMA)
_SENSOR_SLOTS = [(SENSOR_PLAN.leaf(k), 0) for k in (_COUNTS, _ENERGY, _NOISY, _A, _B, _NA, _NB)]
# record-slot indices of the seven case-study inputs/outputs in the Sensor descriptor (plan order)
_FUSED_FIELDS = [[lf.dotted for lf, _, _, _ in cv._slot_table(SENSOR_PLAN)].index(k)
                 for k in (_COUNTS, _ENERGY, _NOISY, _A, _B, _NA, _NB)]
