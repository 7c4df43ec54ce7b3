"""CPU baseline legs of bench.py (TEST / BASELINE INFRASTRUCTURE ONLY).

The reference's own conversion path, restated on numpy so it runs on the GPU
box without /root/reference: per leaf, a strided column view of the packed
struct, np.ascontiguousarray (the gather) and a byte copy into the plane
(transfer.py:196-228). Timed with the reference protocol: warm-up, then the
mean of the fastest samples (bench.py:214-215).
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os
import time

import numpy as np

OBJ8 = np.dtype([(f"f{i}", "<f4" if i % 2 == 0 else "<i4") for i in range(8)])


def per_leaf_convert(records: np.ndarray, planes: list[np.ndarray]) -> None:
    """transfer.py:203-205 (column), 226 (ascontiguousarray), 228 (copy into plane)."""
    for name, plane in zip(records.dtype.names, planes):
        packed = np.ascontiguousarray(records[name])
        plane.view(np.uint8)[:] = packed.view(np.uint8).reshape(-1)


def mean_of_fastest(samples, keep: int) -> float:
    return sum(sorted(samples)[:keep]) / keep


def single_core(n: int, budget_s: float = 15.0, seed: int = 1) -> dict:
    """Reference path on one core: objects/s and GB/s (64 B/object algorithmic)."""
    rng = np.random.default_rng(seed)
    rec = np.frombuffer(rng.integers(0, 256, n * 32, dtype=np.uint8).tobytes(), OBJ8)
    planes = [np.empty(n, OBJ8[i]) for i in range(8)]
    per_leaf_convert(rec, planes)  # warm-up
    samples = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(samples) < 3:
        t0 = time.perf_counter()
        per_leaf_convert(rec, planes)
        samples.append(time.perf_counter() - t0)
    t = mean_of_fastest(samples, max(1, min(10, len(samples) // 3)))
    return {"seconds": t, "objects_per_s": n / t, "gbs": n * 64 / t / 1e9, "reps": len(samples)}


# ---- multi-core arm ----------------------------------------------------------------------

_G = {}


def _work(span):
    lo, hi = span
    per_leaf_convert(_G["rec"][lo:hi], [pl[lo:hi] for pl in _G["planes"]])
    return hi - lo


def multi_core(n: int, steps: int, warmup: int, procs: int | None = None, seed: int = 1) -> dict:
    """The reference path sharded over all host cores (one process per core).
    Buffers are anonymous shared mappings inherited through fork, so a small
    /dev/shm does not matter."""
    procs = procs or os.cpu_count() or 1
    a = mmap.mmap(-1, n * 32)
    p = mmap.mmap(-1, n * 32)
    try:
        rec = np.frombuffer(a, OBJ8)
        rng = np.random.default_rng(seed)
        chunk = 1 << 24
        for lo in range(0, n * 32, chunk):
            hi = min(lo + chunk, n * 32)
            np.frombuffer(a, np.uint8)[lo:hi] = rng.integers(0, 256, hi - lo, dtype=np.uint8)
        base = np.frombuffer(p, np.uint8)
        _G["rec"] = rec
        _G["planes"] = [base[i * n * 4 : (i + 1) * n * 4].view(OBJ8[i]) for i in range(8)]
        cuts = np.linspace(0, n, procs * 4 + 1).astype(np.int64)
        spans = list(zip(cuts[:-1].tolist(), cuts[1:].tolist()))
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            for _ in range(warmup):
                pool.map(_work, spans)
            times = []
            for _ in range(steps):
                t0 = time.perf_counter()
                done = sum(pool.map(_work, spans))
                times.append(time.perf_counter() - t0)
                assert done == n
        # the children wrote through the shared mapping: spot-check one plane
        assert np.array_equal(_G["planes"][3][: min(n, 1000)], rec["f3"][: min(n, 1000)])
        return {"step_seconds": times, "procs": procs, "n": n}
    finally:
        _G.clear()
        del rec, base
        a.close()
        p.close()


# ---- per-config single-core legs (bench extras) ------------------------------------------

def _rate(fn, budget_s: float) -> float:
    """seconds per call: warm-up, then the mean of the fastest third (bench.py:214-215)"""
    fn()
    samples = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(samples) < 3:
        t0 = time.perf_counter()
        fn()
        samples.append(time.perf_counter() - t0)
    return mean_of_fastest(samples, max(1, min(10, len(samples) // 3)))


def per_config(budget_s: float = 2.0, seed: int = 3) -> dict:
    """The reference's CPU path for configs 1-4 on one core, on bounded samples
    of each workload (rates scale linearly in the sample size):
    1: per-leaf AoS->planes of 1M Obj8 (transfer.py:196-228);
    2: one 436x436 event, per-leaf AoS->planes of the 30 B Sensor record, then
       calibrate + noise (detector/schemas.py:29-41);
    3: jagged_fill of 100K clusters from a shuffled pool: per-segment
       np.asarray + concatenate + cumsum (collection.py:537-556);
    4: 1M Track records -> AoSoA T=128 of [pz, px, x, charge] with numpy casts."""
    from . import restate as R

    rng = np.random.default_rng(seed)
    out = {}
    n1 = 1_000_000
    rec = np.frombuffer(rng.integers(0, 256, n1 * 32, dtype=np.uint8).tobytes(), OBJ8)
    planes = [np.empty(n1, OBJ8[i]) for i in range(8)]
    t = _rate(lambda: per_leaf_convert(rec, planes), budget_s)
    out["config1_obj8"] = {"sample": f"{n1} objects", "objects_per_s": n1 / t, "gbs": n1 * 64 / t / 1e9}

    ev = R.generate_event(436, 436, seed=0, density=0.002)
    aos = R.sensor_aos(ev)
    cal = aos["calibration_data"]
    cols = {"type": aos["type"], "counts": aos["counts"], "energy": aos["energy"],
            **{k: cal[k] for k in cal.dtype.names}}  # the 8 leaves, plan order
    cells = aos.size
    splanes = {k: np.empty(cells, v.dtype) for k, v in cols.items()}

    def case_study():
        for k, v in cols.items():
            splanes[k][:] = np.ascontiguousarray(v)
        e = R.calibrate(splanes["counts"], splanes["parameter_A"], splanes["parameter_B"])
        R.noise(e, splanes["noise_A"], splanes["noise_B"], splanes["noisy"])

    t = _rate(case_study, budget_s)
    out["config2_sensor"] = {"sample": f"1 event, {cells} cells", "cells_per_s": cells / t,
                             "gbs": cells * 64 / t / 1e9}

    n3 = 100_000
    lens = rng.integers(0, 21, n3).astype(np.int32)
    order = rng.permutation(n3)
    gaps = lens[order].astype(np.int64) + rng.integers(0, 4, n3)
    offs = np.empty(n3, np.int64)
    offs[order] = np.concatenate([[0], np.cumsum(gaps)[:-1]])
    pool = rng.integers(0, 1 << 62, int(gaps.sum()), dtype=np.uint64)
    segments = [pool[o:o + n] for o, n in zip(offs.tolist(), lens.tolist())]  # the caller's per-object vectors
    members = int(lens.sum())

    def jagged_fill():
        arrs = [np.asarray(s, dtype=np.uint64) for s in segments]
        pv = np.zeros(n3 + 1, np.int32)
        pv[1:] = np.cumsum(np.array([a.size for a in arrs], np.int64)).astype(np.int32)
        np.concatenate(arrs)

    t = _rate(jagged_fill, budget_s)
    out["config3_jagged"] = {"sample": f"{n3} clusters, {members} members", "members_per_s": members / t,
                             "gbs": (n3 * 16 + members * 16) / t / 1e9}

    n4 = 1_000_000
    track = np.dtype([("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("px", "<f8"), ("py", "<f8"), ("pz", "<f8"),
                      ("charge", "<i4"), ("id", "<u8")])
    trk = np.frombuffer(rng.integers(0, 256, n4 * 60, dtype=np.uint8).tobytes(), track)
    fields = [("pz", "f32"), ("px", "f32"), ("x", "f32"), ("charge", "i32")]
    with np.errstate(all="ignore"):
        t = _rate(lambda: R.to_aosoa(trk, fields, 128), budget_s)
    out["config4_aosoa"] = {"sample": f"{n4} tracks", "objects_per_s": n4 / t, "gbs": n4 * 76 / t / 1e9}
    return out


# ---- the reference package itself (baseline/_ref) ------------------------------------------

def import_reference():
    """soakit from the git-ignored install under baseline/_ref (it travels to the
    GPU box); None when it is absent -- the callers then time the port above."""
    import importlib
    import sys

    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(root, "soakit")):
        return None
    if root not in sys.path:
        sys.path.append(root)
    return importlib.import_module("soakit")


def _soakit_pair(sk, n: int, seed: int):
    """AoS source with random records and a per_field destination, both host
    collections of the Obj8 schema (8 x f32/i32)."""
    schema = sk.Schema("Obj8", tuple(sk.declare_per_item(f"f{i}", sk.F32 if i % 2 == 0 else sk.I32)
                                     for i in range(8)))
    src = sk.Collection(schema, "aos")
    src.resize(n)
    rng = np.random.default_rng(seed)
    raw = src.layout._struct_buf._data
    chunk = 1 << 24
    for lo in range(0, n * 32, chunk):
        hi = min(lo + chunk, n * 32)
        raw[lo:hi] = rng.integers(0, 256, hi - lo, dtype=np.uint8)
    return src, sk.Collection(schema, "per_field")


def reference_single_core(n: int, budget_s: float = 12.0, seed: int = 1) -> dict | None:
    """soakit's own copy_collection(per_field, aos) on host collections
    (per-leaf-default, transfer.py:171-236), one core, reference protocol."""
    sk = import_reference()
    if sk is None:
        return None
    src, dst = _soakit_pair(sk, n, seed)
    assert sk.transfer.copy_collection(dst, src) == "per-leaf-default"
    t = _rate(lambda: sk.transfer.copy_collection(dst, src), budget_s)
    return {"seconds": t, "objects_per_s": n / t, "gbs": n * 64 / t / 1e9, "kind": "reference"}


def _ref_worker(span, seed, steps, start, done, out):
    sk = import_reference()
    src, dst = _soakit_pair(sk, span, seed)
    sk.transfer.copy_collection(dst, src)  # warm-up, also sizes dst
    for _ in range(steps):
        start.wait()
        sk.transfer.copy_collection(dst, src)
        done.wait()
    out.put(int(dst.size()))


def reference_multi_core(n: int, steps: int, warmup: int, procs: int | None = None, seed: int = 1) -> dict | None:
    """soakit's copy_collection on every host core: one process per core owns
    a contiguous 1/procs shard (its own AoS and per_field collections); a step
    is every shard converting once, timed by the parent between two barriers."""
    if import_reference() is None:
        return None
    procs = procs or os.cpu_count() or 1
    cuts = np.linspace(0, n, procs + 1).astype(np.int64)
    ctx = mp.get_context("fork")
    total = steps + warmup
    start, done = ctx.Barrier(procs + 1), ctx.Barrier(procs + 1)
    out = ctx.Queue()
    workers = [ctx.Process(target=_ref_worker, args=(int(cuts[i + 1] - cuts[i]), seed + i, total, start, done, out))
               for i in range(procs)]
    for w in workers:
        w.start()
    times = []
    try:
        for k in range(total):
            start.wait()
            t0 = time.perf_counter()
            done.wait()
            if k >= warmup:
                times.append(time.perf_counter() - t0)
        converted = sum(out.get(timeout=60) for _ in workers)
        assert converted == n
    finally:
        for w in workers:
            w.join(timeout=60)
    return {"step_seconds": times, "procs": procs, "n": n, "kind": "reference"}


def reference_per_config(budget_s: float = 2.0, seed: int = 3) -> dict | None:
    """Configs 1-3 through soakit itself (baseline/_ref), one core, on bounded
    samples, timed with the reference protocol:
    1: copy_collection(per_field, aos) of 1M Obj8 on the host (per-leaf-default);
    2: one 436x436 event: fill_sensor_collection into a host AoS collection
       (untimed), copy_collection(per_field@mockdev, aos@host) +
       calibrate_collection + noise_for_collection inside execution_scope("mockdev");
    3: Collection.jagged_fill of 100K clusters from per-object segments.
    Config 4 (AoSoA/cast) has no reference path: the port's figure stays.
    None when soakit is absent."""
    sk = import_reference()
    if sk is None:
        return None
    from soakit.detector import events as ev
    from soakit.detector import reconstruct as rc
    from soakit.detector import schemas as ds

    rng = np.random.default_rng(seed)
    out = {}
    n1 = 1_000_000
    src, dst = _soakit_pair(sk, n1, seed)
    t = _rate(lambda: sk.transfer.copy_collection(dst, src), budget_s)
    out["config1_obj8"] = {"sample": f"{n1} objects, soakit copy_collection(per_field, aos)",
                           "objects_per_s": n1 / t, "gbs": n1 * 64 / t / 1e9}

    event = ev.generate_event(ev.EventSpec(436, 436, 0, 0.002))
    host_pf = sk.Collection(ds.SENSOR_SCHEMA, "per_field")
    rc.fill_sensor_collection(host_pf, event)
    host = sk.Collection(ds.SENSOR_SCHEMA, "aos")
    sk.transfer.copy_collection(host, host_pf)
    cells = host.size()
    sk.memctx.configure_mockdev(capacity_bytes=1 << 30)
    dev = sk.Collection(ds.SENSOR_SCHEMA, "per_field", sk.memctx.ContextInfo.mockdev())

    def case_study():
        sk.transfer.copy_collection(dev, host)
        with sk.memctx.execution_scope("mockdev"):
            ds.calibrate_collection(dev)
            ds.noise_for_collection(dev)

    t = _rate(case_study, budget_s)
    out["config2_sensor"] = {"sample": f"1 event, {cells} cells, soakit per-leaf AoS@host -> per_field@mockdev "
                                       "+ calibrate + noise", "cells_per_s": cells / t, "gbs": cells * 64 / t / 1e9}

    # the second phase of the case study (bench.py:180-184): reconstruct one calibrated event
    with sk.memctx.execution_scope("mockdev"):
        energy = dev.column("energy").read().copy()
        noise = ds.noise_for_collection(dev)
        stype = dev.column("type").read().copy()
        noisy = dev.column("calibration_data.noisy").read().copy()
    t = _rate(lambda: rc.reconstruct_arrays(energy, noise, stype, noisy, 436, 436), budget_s)
    out["config2_reconstruct"] = {"sample": "1 event 436x436, soakit reconstruct_arrays",
                                  "events_per_s": 1.0 / t, "ms_per_event": t * 1e3}

    n3 = 100_000
    lens = rng.integers(0, 21, n3)
    pool = rng.integers(0, 1 << 62, int(lens.sum()), dtype=np.uint64)
    cuts = np.concatenate([[0], np.cumsum(lens)])
    order = rng.permutation(n3)
    segments = [pool[cuts[i]:cuts[i + 1]] for i in order]  # per-object vectors in shuffled memory order
    schema = sk.Schema("Cluster", (sk.declare_per_item("seed", sk.U64), sk.declare_jagged("members", sk.I32, sk.U64)))
    coll = sk.Collection(schema, "per_field")
    coll.resize(n3)
    members = int(lens.sum())
    t = _rate(lambda: coll.jagged_fill("members", segments), budget_s)
    out["config3_jagged"] = {"sample": f"{n3} clusters, {members} members, soakit Collection.jagged_fill",
                             "members_per_s": members / t, "gbs": (n3 * 16 + members * 16) / t / 1e9}
    for v in out.values():
        v["kind"] = "reference"
    return out
