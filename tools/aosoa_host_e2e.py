import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, workloads as wl, schema as sc
from oracle import restate
n = 16_000_000
pin = mc.ContextInfo.pinned()
a = sk.Collection(wl.TRACK_SCHEMA, ly.AOS, pin)
a.reserve(n)
with a.layout.engine_ops():
    a.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
recs = wl.track_records(n)
a.layout._struct_buf._data[: n * 60] = recs.view(np.uint8)
fields = [sk.AosoaField("pz", "f32"), sk.AosoaField("px", "f32"), sk.AosoaField("x", "f32"), sk.AosoaField("charge", "i32")]
ao = sk.Aosoa(n, 128, fields, mc.ContextInfo.cuda(0))
sk.to_aosoa(a, fields, 128, out=ao)
t0 = time.perf_counter()
for _ in range(5):
    sk.to_aosoa(a, fields, 128, out=ao)
dt = (time.perf_counter() - t0) / 5
print("pinned AoS -> device AoSoA", round(dt * 1e3, 3), "ms", round(n * 60 / dt / 1e9, 1), "GB/s H2D")
got = np.empty(ao.tile_bytes, np.uint8)
nat.memcpy(got.ctypes.data, ao.buffer.ptr, ao.tile_bytes, 0); nat.sync(0)
want = restate.to_aosoa(recs[:128], [(f.leaf, f.dtype) for f in fields], 128, ao.tile_bytes)
print("tile 0 ok", got.tobytes() == bytes(want))
