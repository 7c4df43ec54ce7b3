import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat, jagged, layouts as ly, memctx as mc, workloads as wl
from paper_2511_04853_b200.devarray import DeviceArray
CUDA = mc.ContextInfo.cuda(0)
for n in (16, 1_000_000):
    lens, offsets, pool = wl.cluster_inputs(n, seed=7)
    d = [DeviceArray.from_numpy(x, CUDA) for x in (lens, offsets, pool)]
    c = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.resize(n)
    for _ in range(5): jagged.pack(c, "members", *d)
    t0 = time.perf_counter()
    for _ in range(50): jagged.pack(c, "members", *d)
    print(f"n={n}: {1e6*(time.perf_counter()-t0)/50:.1f} us/pack")
pr = cProfile.Profile(); pr.enable()
for _ in range(50): jagged.pack(c, "members", *d)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(10)
