"""Collection.jagged_fill of 1M clusters from per-object numpy segments (the reference's API) on a device
collection: host packing + H2D + GPU pack, wall time; and the reference's own jagged_fill on the host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import layouts as ly, memctx as mc, workloads as wl  # noqa: E402

n = 1_000_000
rng = np.random.default_rng(7)
lens = rng.integers(0, 21, n)
pool = rng.integers(0, 2**63, int(lens.sum()), dtype=np.uint64)
cuts = np.concatenate([[0], np.cumsum(lens)])
segs = [pool[cuts[i]:cuts[i + 1]] for i in rng.permutation(n)]
c = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(0))
with mc.execution_scope(mc.CUDA):
    c.resize(n)
    for _ in range(2):
        c.jagged_fill("members", segs)
    t = []
    for _ in range(5):
        t0 = time.perf_counter()
        c.jagged_fill("members", segs)
        t.append(time.perf_counter() - t0)
print(f"jagged_fill 1M clusters (device collection): {min(t) * 1e3:.1f} ms (best of 5)")

from paper_2511_04853_b200 import _segpack, jagged  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402


def best(fn, k=5):
    r = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        r.append(time.perf_counter() - t0)
    return min(r) * 1e3


print(f"  segpack: {best(lambda: _segpack.pack_segments(segs, np.uint64)):.1f} ms")
ob = np.frombuffer(_segpack.pack_segments(segs, np.uint64), np.uint8)
L = ob[:8 * n].view(np.int64)
P = ob[16 * n:].view(np.uint64)
S = np.zeros(n, np.int64)
print(f"  cumsum: {best(lambda: np.cumsum(L[:-1], out=S[1:])):.1f} ms")
with mc.execution_scope(mc.CUDA):
    print(f"  pack pageable: {best(lambda: jagged.pack(c, 'members', L, S, P)):.1f} ms")
    pins = []
    for a in (L, S, P):
        b = mc.allocate(mc.ContextInfo.pinned(), a.nbytes)
        v = np.frombuffer(b._data, a.dtype, a.size)
        v[:] = a
        pins.append(v)
    print(f"  pack pinned: {best(lambda: jagged.pack(c, 'members', *pins)):.1f} ms")
    ds = [DeviceArray.from_numpy(a, mc.ContextInfo.cuda(0)) for a in (L, S, P)]
    print(f"  pack device inputs: {best(lambda: jagged.pack(c, 'members', *ds)):.1f} ms")
    print(f"  device alloc+free 88MB: "
          f"{best(lambda: DeviceArray(P.size, np.uint64, mc.ContextInfo.cuda(0)).free()):.2f} ms")
    tmp = np.empty_like(P)
    print(f"  memcpy pool host->host: {best(lambda: np.copyto(tmp, P)):.1f} ms")


from oracle.cpu_baseline import import_reference  # noqa: E402

ref = import_reference()
if ref is not None:
    schema = ref.Schema("Cluster", (ref.declare_per_item("seed", ref.U64),
                                    ref.declare_jagged("members", ref.I32, ref.U64)))
    rc = ref.Collection(schema, "per_field")
    rc.resize(n)
    t0 = time.perf_counter()
    rc.jagged_fill("members", segs)
    print(f"reference jagged_fill 1M clusters (soakit, host): {(time.perf_counter() - t0) * 1e3:.1f} ms")
