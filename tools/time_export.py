"""Breakdown of export_particles_from_collection after a 64-event reconstruction:
the K2 conversion into pinned AoS (copy_collection), the host copies of the
records / pool / prefix, and the per-particle views."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, _segpack, layouts as ly, memctx as mc, sensor  # noqa: E402
from paper_2511_04853_b200.transfer import copy_collection  # noqa: E402

cuda = mc.ContextInfo.cuda(0)
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cuda)
sensor.generate_events(gen, 436, 436, range(64), 0.002, sync=True)
sensor.calibrate_collection(gen)
noise = sensor.noise_for_collection(gen, sync=True)
parts = sensor.reconstruct_from_collection(gen, 436, 436, events=64, noise=noise)
stage = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, mc.ContextInfo.pinned())


def t(fn, reps=10):
    fn()
    nat.sync(0)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    nat.sync(0)
    return (time.perf_counter() - t0) / reps * 1e3


res = {"particles": len(parts)}
res["copy_collection_ms"] = t(lambda: copy_collection(stage, parts))
n = stage.size()
lay = stage.layout
res["recs_copy_ms"] = t(lambda: np.array(lay._struct_buf._data[: n * sensor.PARTICLE_AOS_DTYPE.itemsize]
                                         .view(sensor.PARTICLE_AOS_DTYPE)))
pool = np.array(lay._plane_view(stage.plan.leaf("sensors.value"), 0))
res["pool_copy_ms"] = t(lambda: np.array(lay._plane_view(stage.plan.leaf("sensors.value"), 0)))
b = np.array(lay._plane_view(stage.plan.leaf("sensors.prefix_sum"), 0)).astype(np.int64)
res["split_views_ms"] = t(lambda: _segpack.split_views(pool, b[: n + 1]))
res["export_total_ms"] = t(lambda: sensor.export_particles_from_collection(parts, stage))
res["pool_members"] = int(pool.size)
res["reco_ms"] = t(lambda: sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise), 5)
res["reco_plus_export_ms"] = t(lambda: (sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64,
                                                                            noise=noise),
                                        sensor.export_particles_from_collection(parts, stage)), 5)
raw = lay._struct_buf._data
res["recs_bytecopy_ms"] = t(lambda: np.array(raw[: n * sensor.PARTICLE_AOS_DTYPE.itemsize]).view(sensor.PARTICLE_AOS_DTYPE))
print({k: round(v, 3) if isinstance(v, float) else v for k, v in res.items()})
