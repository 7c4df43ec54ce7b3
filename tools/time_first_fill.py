"""jagged.pack into a FRESH device collection (pool capacity 0: prefix + validation in one launch, grow,
gather) against a repeat fill (capacity already there: one fused launch), config 3 shape, device inputs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, jagged, layouts as ly, memctx as mc, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
lens, offsets, pool = wl.cluster_inputs(1_000_000, seed=7)
d = [DeviceArray.from_numpy(x, CUDA) for x in (lens, offsets, pool)]


def fresh():
    c = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.resize(1_000_000)
    nat.sync(0)
    t0 = time.perf_counter()
    jagged.pack(c, "members", *d)
    dt = time.perf_counter() - t0
    return c, dt


c, _ = fresh()
c.free()
ts = []
for _ in range(10):
    c, dt = fresh()
    ts.append(dt)
    c.free()
c, _ = fresh()
rep = []
for _ in range(10):
    t0 = time.perf_counter()
    jagged.pack(c, "members", *d)
    rep.append(time.perf_counter() - t0)
print({"first_fill_ms": round(min(ts) * 1e3, 3), "repeat_fill_ms": round(min(rep) * 1e3, 3)})
