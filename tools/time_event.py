"""Per-event host overhead of the case-study transfer (one 436x436 event from pinned AoS):
wall time of transfer_calibrate / copy_collection, with a cProfile of the fused call."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, sensor, transfer as tr  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

ev = 436 * 436
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(0))
sensor.generate_events(gen, 436, 436, range(1), 0.002, sync=True)
src = sk.Collection(sensor.SENSOR_SCHEMA, ly.AOS, mc.ContextInfo.pinned())
tr.copy_collection(src, gen)
d1 = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(0))
n1 = DeviceArray(ev, np.float32, mc.ContextInfo.cuda(0))


def best(fn, reps=50):
    fn()
    s = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        s.append(time.perf_counter() - t0)
    return sum(sorted(s)[:10]) / 10 * 1e3


res = {"fused_ms": best(lambda: sensor.transfer_calibrate(d1, src, n1)),
       "copy_only_ms": best(lambda: tr.copy_collection(d1, src)),
       "h2d_only_ms": best(lambda: (nat.memcpy(n1.ptr, src.layout._struct_buf.ptr, ev * 4, 0), nat.sync(0))),
       "h2d_full_event_ms": None}
tmp = DeviceArray(ev * 30 // 4 + 1, np.float32, mc.ContextInfo.cuda(0))
res["h2d_full_event_ms"] = best(lambda: (nat.memcpy(tmp.ptr, src.layout._struct_buf.ptr, ev * 30, 0), nat.sync(0)))
print({k: round(v, 4) for k, v in res.items()})
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    sensor.transfer_calibrate(d1, src, n1)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    tr.copy_collection(d1, src)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
