"""Device time (queued behind a fill) of the fused case study (config 2: 64
generated events, AoS -> planes + energy + noise), for tile sweeps:
SK_TILE_BYTES=... SK_CTAS=... python tools/time_sensor.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, schema as sc  # noqa: E402
from paper_2511_04853_b200 import sensor, transfer as tr  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

cuda = mc.ContextInfo.cuda(0)
busy = DeviceArray(6 << 30, np.uint8, cuda)


def coll(schema, kind, n):
    c = sk.Collection(schema, kind, cuda)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    return c


cells = 64 * 436 * 436
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cuda)
sensor.generate_events(gen, 436, 436, range(64), 0.002, sync=True)
a = coll(sensor.SENSOR_SCHEMA, ly.AOS, cells)
tr.copy_collection(a, gen)
p = coll(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cells)
noise = DeviceArray(cells, np.float32, cuda)
res = []
for rep in range(3):
    for _ in range(3):
        sensor.transfer_calibrate(p, a, noise, sync=False)
    nat.sync(0)
    e0, e1 = nat.Event(), nat.Event()
    nat.call("sk_fill_random", busy.ptr, busy.n, 1, 0, nat.stream(0))
    e0.record(0)
    for _ in range(10):
        sensor.transfer_calibrate(p, a, noise, sync=False)
    e1.record(0)
    nat.sync(0)
    res.append(e0.elapsed_ms(e1) / 10)
print(os.environ.get("SK_TILE_BYTES", "default"), os.environ.get("SK_CTAS", "-"),
      [round(x * 1e3, 1) for x in res], "us; GB/s", round(cells * 64 / min(res) / 1e6))


def queued(fn, reps=10):
    for _ in range(3):
        fn()
    nat.sync(0)
    e0, e1 = nat.Event(), nat.Event()
    nat.call("sk_fill_random", busy.ptr, busy.n, 1, 0, nat.stream(0))
    e0.record(0)
    for _ in range(reps):
        fn()
    e1.record(0)
    nat.sync(0)
    return e0.elapsed_ms(e1) / reps


# the same real events through the plain conversion (no case-study epilogue), both directions
for name, fn in (("a2p", lambda: tr.copy_collection(p, a, {"async": True})),
                 ("p2a", lambda: tr.copy_collection(a, p, {"async": True}))):
    ms = queued(fn)
    print(f"plain {name}: {ms * 1e3:.1f} us, {cells * 60 / ms / 1e6:.0f} GB/s ({cells * 60 / ms / 1e6 / 6546.9:.3f})")
