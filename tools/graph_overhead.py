"""Wall-clock per repeated transfer: copy_collection vs a prepared (CUDA-graph)
transfer, for small device-resident and pinned-host Obj8 conversions."""

import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import layouts as ly, transfer as tr, workloads as wl  # noqa: E402

CUDA = sk.ContextInfo.cuda(0)
PINNED = sk.ContextInfo.pinned()


def timeit(fn, reps=2000):
    for _ in range(50):
        fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps * 1e6


out = []
for n in (1_000, 100_000, 2_000_000):
    for where in ("cuda", "pinned"):
        src = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, PINNED)
        src.resize(n)
        src.layout._struct_buf._data[: n * 32] = np.random.default_rng(0).integers(0, 256, n * 32, dtype=np.uint8)
        if where == "cuda":
            d = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
            tr.copy_collection(d, src)
            src = d
        dst = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
        prep = tr.prepare(dst, src)
        reps = 2000 if n < 1e6 else 200
        a = timeit(lambda: tr.copy_collection(dst, src), reps)
        b = timeit(lambda: prep.run(), reps)
        out.append({"n": n, "src": where, "copy_collection_us": round(a, 2), "prepared_us": round(b, 2)})
        print(json.dumps(out[-1]), flush=True)
        prep.close()
