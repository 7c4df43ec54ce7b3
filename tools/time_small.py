"""Device time (queued behind a fill) of Obj8 AoS->SoA at small N, for tile-size sweeps:
SK_TILE_BYTES=... python tools/time_small.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, schema as sc  # noqa: E402
from paper_2511_04853_b200 import transfer as tr, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
busy = DeviceArray(6 << 30, np.uint8, CUDA)


def coll(kind, n):
    c = sk.Collection(wl.OBJ8_SCHEMA, kind, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    return c


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
    return a.elapsed_ms(b) / steps * 1e3


res = {}
for n in (100_000, 1_000_000, 4_000_000):
    a, p = coll(ly.AOS, n), coll(ly.PER_FIELD, n)
    wl.fill_random_device(a.layout._struct_buf.ptr, n * 32, 1, 0)
    res[n] = round(queued(lambda: tr.copy_collection(p, a, {"async": True})), 2)
    a.free()
    p.free()
print(os.environ.get("SK_TILE_BYTES", "default"), os.environ.get("SK_CTAS", "-"), res)
