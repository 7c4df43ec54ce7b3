"""Host timeline of reconstruct_from_collection (64 events): wall time at each step, no extra syncs."""
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
marks = {}
orig_call, orig_sync = nat.call, nat.sync
t_start = [0.0]


def mark(name):
    marks[name] = marks.get(name, 0.0) + (time.perf_counter() - t_start[0]) * 1e6


def call(name, *a):
    r = orig_call(name, *a)
    mark("after " + name)
    return r


def sync(dev):
    mark("before sync")
    orig_sync(dev)
    mark("after sync")


for _ in range(5):
    sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise)
nat.call, nat.sync = call, sync
reps = 20
for _ in range(reps):
    t_start[0] = time.perf_counter()
    sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise)
    mark("return")
nat.call, nat.sync = orig_call, orig_sync
for k, v in sorted(marks.items(), key=lambda kv: kv[1]):
    print(f"{v / reps:8.1f} us  {k}")
