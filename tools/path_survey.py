"""Device GB/s of every conversion pair on the workload schemas (queued behind a
fill, events on the library stream): AoS<->planes for Obj8 / Sensor / Particle /
Track, and AoSoA in both directions from both sides. Algorithmic bytes = bytes
read + bytes written once. Prints one JSON line per path."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, schema as sc, sensor  # noqa: E402
from paper_2511_04853_b200 import transfer as tr, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
busy = DeviceArray(6 << 30, np.uint8, CUDA)
PEAK = 6551.7


def coll(schema, kind, n):
    c = sk.Collection(schema, kind, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    for b in c.layout.buffers():
        if b.length_bytes:
            wl.fill_random_device(b.ptr, b.length_bytes // 8 * 8, 7, 0)
    return c


def queued(fn, steps=8):
    for _ in range(2):
        fn()
    nat.sync(0)
    a, b = nat.Event(), nat.Event()
    nat.call("sk_fill_random", busy.ptr, busy.n, 1, 0, nat.stream(0))
    a.record(0)
    for _ in range(steps):
        fn()
    b.record(0)
    nat.sync(0)
    return a.elapsed_ms(b) / steps


def report(name, ms, nbytes, extra=None):
    gbs = nbytes / ms / 1e6
    print(json.dumps({"path": name, "ms": round(ms, 4), "gbs": round(gbs, 1), "frac": round(gbs / PEAK, 3),
                      **(extra or {})}), flush=True)


def main_bytes(c):
    return sum(lf.value_type.size_bytes * lf.extent_multiplier for lf in c.plan.leaves
               if lf.size_tag == sc.MAIN_TAG and lf.role == "element")


schemas = {"obj8": (wl.OBJ8_SCHEMA, 60_000_000), "sensor": (sensor.SENSOR_SCHEMA, 60_000_000),
           "particle": (sensor.PARTICLE_SCHEMA, 30_000_000), "track": (wl.TRACK_SCHEMA, 30_000_000)}
only = os.environ.get("PATHS")
for name, (schema, n) in schemas.items():
    if only and name not in only.split(","):
        continue
    a, p = coll(schema, ly.AOS, n), coll(schema, ly.PER_FIELD, n)
    rec = main_bytes(a)
    report(f"{name}_aos_to_planes", queued(lambda: tr.copy_collection(p, a, {"async": True})), 2 * n * rec,
           {"record_bytes": rec, "n": n})
    report(f"{name}_planes_to_aos", queued(lambda: tr.copy_collection(a, p, {"async": True})), 2 * n * rec)
    a.free()
    p.free()

if only and "aosoa" not in only.split(","):
    sys.exit(0)
n = 50_000_000
a, p = coll(wl.TRACK_SCHEMA, ly.AOS, n), coll(wl.TRACK_SCHEMA, ly.PER_FIELD, n)
fields = [sk.AosoaField("pz", "f32"), sk.AosoaField("px", "f32"), sk.AosoaField("x", "f32"),
          sk.AosoaField("charge", "i32")]
ao = sk.Aosoa(n, 128, fields, CUDA)
report("track_aos_to_aosoa_cast", queued(lambda: sk.to_aosoa(a, fields, 128, out=ao, sync=False)), n * (60 + 16))
report("track_planes_to_aosoa_cast", queued(lambda: sk.to_aosoa(p, fields, 128, out=ao, sync=False)), n * 44)
full = [sk.AosoaField(f, "f64") for f in ("x", "y", "z", "px", "py", "pz")] + [sk.AosoaField("charge", "i32"),
                                                                               sk.AosoaField("id", "u64")]
ao2 = sk.Aosoa(n, 32, full, CUDA)
report("track_aos_to_aosoa_full", queued(lambda: sk.to_aosoa(a, full, 32, out=ao2, sync=False)), n * 120)
report("track_aosoa_to_aos", queued(lambda: sk.from_aosoa(ao2, a, sync=False)), n * 120)
report("track_aosoa_to_planes", queued(lambda: sk.from_aosoa(ao2, p, sync=False)), n * 120)
