import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import convert as cv, layouts as ly, memctx as mc, schema as sc, sensor, workloads as wl
import ctypes as C
from paper_2511_04853_b200 import _native as nat
CUDA = mc.ContextInfo.cuda(0)
def coll(schema, kind, n):
    c = sk.Collection(schema, kind, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    return c
for name, schema in [("particle", sensor.PARTICLE_SCHEMA), ("track", wl.TRACK_SCHEMA), ("sensor", sensor.SENSOR_SCHEMA)]:
    a, p = coll(schema, ly.AOS, 1 << 20), coll(schema, ly.PER_FIELD, 1 << 20)
    for d, s, tag in [(p, a, "a2p"), (a, p, "p2a")]:
        desc = cv.plan_desc(d.layout, s.layout, 1 << 20)
        info = cv.plan_info(desc, 0)
        ok = C.c_int(0); buf = C.create_string_buffer(1 << 16); ln = C.c_size_t(0)
        rc = nat.lib().sk_convert_specialize_check(C.byref(desc), C.byref(ok), buf, len(buf), C.byref(ln))
        print(name, tag, json.dumps(info), "specialised" if ok.value else "generic", "nfields", desc.nfields)
