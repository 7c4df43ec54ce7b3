"""Device GB/s of a few record signatures through copy_collection (100M-class sizes, back-to-back launches):
Sensor AoS->planes (30 B), Particle AoS->planes (64 B, byte fields), Track AoS->planes (60 B), and back."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.profile_one import coll  # noqa: E402
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, sensor, transfer as tr, workloads as wl  # noqa: E402

PEAK = 6546.9
cases = [("sensor", sensor.SENSOR_SCHEMA, 30, 64 * 436 * 436), ("particle", sensor.PARTICLE_SCHEMA, 64, 50_000_000),
         ("track", wl.TRACK_SCHEMA, 60, 100_000_000)]
only = os.environ.get("CASES")
for name, schema, stride, n in cases:
    if only and name not in only.split(","):
        continue
    a, p = coll(schema, ly.AOS, n), coll(schema, ly.PER_FIELD, n)
    wl.fill_random_device(a.layout._struct_buf.ptr, n * stride // 8 * 8, 5, 0)
    for direction, fn in (("a2p", lambda: tr.copy_collection(p, a, {"async": True})),
                          ("p2a", lambda: tr.copy_collection(a, p, {"async": True}))):
        for _ in range(3):
            fn()
        nat.sync(0)
        e0, e1 = nat.Event(), nat.Event()
        e0.record(0)
        for _ in range(10):
            fn()
        e1.record(0)
        nat.sync(0)
        ms = e0.elapsed_ms(e1) / 10
        gbs = n * stride * 2 / ms / 1e6
        tag = " ".join(f"{v}={os.environ[v]}" for v in ("SK_TILE_BYTES", "SK_STAGES", "SK_SPECIALIZE") if v in os.environ)
        print(f"{name} {direction}: {ms:.3f} ms {gbs:.0f} GB/s frac {gbs / PEAK:.3f} {tag}", flush=True)
    a.free()
    p.free()
