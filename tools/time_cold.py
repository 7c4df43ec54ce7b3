"""Obj8 AoS -> planes device time with a cold L2: rotate over sets of (AoS, planes) pairs whose total
exceeds the 126 MB L2, launches queued behind a device fill. usage: python tools/time_cold.py [n ...]"""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, schema as sc  # noqa: E402
from paper_2511_04853_b200 import transfer as tr, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
PEAK = 6546.9
busy = DeviceArray(4 << 30, np.uint8, CUDA)


def coll(kind, n):
    c = sk.Collection(wl.OBJ8_SCHEMA, kind, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    return c


for n in [int(x) for x in sys.argv[1:]] or [100_000, 1_000_000, 10_000_000]:
    k = max(2, -(-(320 << 20) // (n * 64)))  # pairs so the rotation covers > 320 MB
    sets = []
    for i in range(k):
        a, p = coll(ly.AOS, n), coll(ly.PER_FIELD, n)
        wl.fill_random_device(a.layout._struct_buf.ptr, n * 32, i + 1, 0)
        sets.append((a, p))
    turn = itertools.cycle(sets)

    def step():
        a, p = next(turn)
        tr.copy_collection(p, a, {"async": True})

    for _ in range(2 * k):
        step()
    nat.sync(0)
    steps = 8 * k
    e0, e1 = nat.Event(), nat.Event()
    nat.call("sk_fill_random", busy.ptr, busy.n, 1, 0, nat.stream(0))
    e0.record(0)
    for _ in range(steps):
        step()
    e1.record(0)
    nat.sync(0)
    us = e0.elapsed_ms(e1) / steps * 1e3
    tag = " ".join(f"{v}={os.environ[v]}" for v in ("SK_TILE_BYTES", "SK_STAGES", "SK_CTAS") if v in os.environ)
    print(f"n={n} cold_us={us:.2f} frac={n * 64 / us / 1e3 / PEAK:.3f} {tag}", flush=True)
    for a, p in sets:
        a.free()
        p.free()
