import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, schema as sc, transfer as tr, workloads as wl
CUDA = mc.ContextInfo.cuda(0)
n = int(os.environ.get("N", 1_000_000))
def coll(kind):
    c = sk.Collection(wl.OBJ8_SCHEMA, kind, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    return c
a, p = coll(ly.AOS), coll(ly.PER_FIELD)
wl.fill_random_device(a.layout._struct_buf.ptr, n * 32, 1, 0)
for _ in range(6):
    tr.copy_collection(p, a, {"async": True})
nat.sync(0)
