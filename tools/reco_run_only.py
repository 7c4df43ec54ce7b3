"""sk_reco_run wall time with and without the queued write (64 events)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, sensor  # noqa: E402

cuda = mc.ContextInfo.cuda(0)
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cuda)
sensor.generate_events(gen, 436, 436, range(64), 0.002, sync=True)
sensor.calibrate_collection(gen)
noise = sensor.noise_for_collection(gen, sync=True)
parts = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, cuda)
sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise)
dev, p = sensor._device_planes(gen)
ptype = gen.layout.plane_address(gen.plan.leaf("type"), 0)
out = sensor._reco_out(parts)


def run(with_out):
    h = C.c_void_p(0)
    m, nc, r, wr = C.c_int64(0), C.c_int64(0), C.c_int(0), C.c_int(0)
    nat.call("sk_reco_run", 436, 436, 64, p[sensor._ENERGY], noise.ptr, ptype, p[sensor._NOISY],
             C.byref(out) if with_out else None, 0, nat.stream(0), C.byref(h), C.byref(m), C.byref(nc), C.byref(r),
             C.byref(wr))
    nat.call("sk_reco_free", h, nat.stream(0))


for with_out in (False, True, False, True):
    for _ in range(3):
        run(with_out)
    t0 = time.perf_counter()
    for _ in range(20):
        run(with_out)
    print("with_out" if with_out else "run only", round((time.perf_counter() - t0) / 20 * 1e6, 1), "us")
