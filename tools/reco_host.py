"""Where the host time of reconstruct_from_collection goes (cProfile, 64 events)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, sensor  # noqa: E402

cuda = mc.ContextInfo.cuda(0)
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cuda)
sensor.generate_events(gen, 436, 436, range(64), 0.002, sync=True)
sensor.calibrate_collection(gen)
noise = sensor.noise_for_collection(gen, sync=True)
parts = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, cuda)
for _ in range(3):
    sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    sensor.reconstruct_from_collection(gen, 436, 436, out=parts, events=64, noise=noise)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
