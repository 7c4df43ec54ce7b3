"""Per-call host overhead of copy_collection for small device-resident conversions."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, schema as sc, transfer as tr, workloads as wl
cuda = mc.ContextInfo.cuda(0)
def coll(kind, n):
    c = sk.Collection(wl.OBJ8_SCHEMA, kind, cuda)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    return c
for n in (1000, 1_000_000):
    a, p = coll(ly.AOS, n), coll(ly.PER_FIELD, n)
    for _ in range(50):
        tr.copy_collection(p, a, {"async": True})
    nat.sync(0)
    t0 = time.perf_counter()
    for _ in range(500):
        tr.copy_collection(p, a, {"async": True})
    t1 = time.perf_counter()
    nat.sync(0)
    t2 = time.perf_counter()
    print(f"n={n}: host {1e6*(t1-t0)/500:.1f} us/call, incl. drain {1e6*(t2-t0)/500:.1f} us/call")
pr = cProfile.Profile(); pr.enable()
for _ in range(300):
    tr.copy_collection(p, a, {"async": True})
pr.disable(); nat.sync(0)
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
