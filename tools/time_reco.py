"""Wall time of the phases of reconstruct_from_collection on 64 generated
events (436 x 436, density 0.002): sk_reco_run, sk_reco_write, the jagged pack
of the contributor lists, and the whole call."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, sensor  # noqa: E402

cuda = mc.ContextInfo.cuda(0)
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cuda)
sensor.generate_events(gen, 436, 436, range(64), 0.002, sync=True)
sensor.calibrate_collection(gen)
noise = sensor.noise_for_collection(gen, sync=True)
parts = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, cuda)

calls = {}
orig = nat.call


def timed_call(name, *a):
    t0 = time.perf_counter()
    r = orig(name, *a)
    if name.startswith("sk_reco") or name.startswith("sk_jagged"):
        nat.sync(0)
        calls[name] = calls.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return r


for _ in range(3):
    sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise)
reps = 10
t0 = time.perf_counter()
for _ in range(reps):
    sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise)
total = (time.perf_counter() - t0) * 1e3 / reps
nat.call = timed_call
for _ in range(reps):
    sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise)
nat.call = orig
print({"total_ms": round(total, 3), "particles": len(parts), "rounds": parts.reco_rounds,
       **{k: round(v / reps, 3) for k, v in calls.items()}})
if os.environ.get("STATS"):
    from paper_2511_04853_b200 import layouts as _ly  # noqa: F401
    e = np.frombuffer(bytes(0), np.float32)
    with mc.execution_scope(mc.CUDA):
        e = gen.column("energy").read()
    nz = noise.numpy()
    r = e / nz
    print({"cells": r.size, "seeds(ratio>5)": int((r > 5).sum()), "ratio>2": int((r > 2).sum())})
