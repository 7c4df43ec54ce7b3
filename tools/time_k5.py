"""Device time of the standalone case-study kernels (K5) on 64 generated events (12.2M cells), queued
behind a device fill: calibrate (20 B/cell) and noise (17 B/cell) vs the HBM copy peak."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, sensor  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
PEAK = 6546.9
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
sensor.generate_events(gen, 436, 436, range(64), 0.002)
cells = gen.size()
noise = DeviceArray(cells, np.float32, CUDA)
busy = DeviceArray(4 << 30, np.uint8, CUDA)


def queued(fn, steps=20):
    for _ in range(3):
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


for name, fn, bpc in (("calibrate", lambda: sensor.calibrate_collection(gen, sync=False), 20),
                      ("noise", lambda: sensor.noise_for_collection(gen, noise, sync=False), 17)):
    ms = queued(fn)
    print(f"{name}: {ms * 1e3:.1f} us  {cells * bpc / ms / 1e6:.0f} GB/s  frac {cells * bpc / ms / 1e6 / PEAK:.3f}")
