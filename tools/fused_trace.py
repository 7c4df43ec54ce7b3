"""Per-CTA timeline of the fused jagged pack on config 3 (SK_FUSED_DBG bit 8):
when each CTA knows its block prefix, finishes its blocks and exits."""
import ctypes as C
import os
import sys

os.environ["SK_FUSED_DBG"] = str(int(os.environ.get("SK_FUSED_DBG", "0")) | 8)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2511_04853_b200 import _native as nat, memctx as mc, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
n = int(os.environ.get("N", 1_000_000))
lens, offsets, pool = wl.cluster_inputs(n, seed=7)
T = int(lens.sum())
d_lens, d_off, d_pool = (DeviceArray.from_numpy(x, CUDA) for x in (lens, offsets, pool))
prefix = DeviceArray(n + 1, np.int32, CUDA)
need = C.c_size_t(0)
nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
scratch = DeviceArray(need.value, np.uint8, CUDA)
total = DeviceArray(2, np.int64, CUDA)
out = DeviceArray(T + 1000, np.uint64, CUDA)
I32 = nat.TYPE_CODES["i32"]
foff, fsz, dst = (C.c_int64 * 1)(0), (C.c_int32 * 1)(8), (C.c_void_p * 1)(out.ptr)
for _ in range(6):
    nat.call("sk_jagged_pack", n, d_lens.ptr, I32, prefix.ptr, I32, d_off.ptr, d_pool.ptr, pool.size, 8, 1, foff,
             fsz, dst,
             T + 1000, scratch.ptr, scratch.n, total.ptr, nat.stream(0))
buf = np.zeros(1024 * 8, np.uint64)
nat.call("sk_jagged_trace", buf.ctypes.data, buf.nbytes)
t = buf.reshape(1024, 8).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
spins = t[:, 7].copy()
t[:, 7] = t[:, 0]
rel = (t - t0) / 1e3
print("pred-sum polling rounds: p50", np.percentile(spins, 50), "max", spins.max())
for k, name in [(0, "start"), (4, "total out"), (6, "first poll back"), (5, "preds summed"), (1, "prefix known"),
                (2, "blocks done"), (3, "exit")]:
    q = np.percentile(rel[:, k], [0, 10, 50, 90, 100])
    print(f"{name:13s} us: min {q[0]:6.2f}  p10 {q[1]:6.2f}  p50 {q[2]:6.2f}  p90 {q[3]:6.2f}  max {q[4]:6.2f}")
if os.environ.get("PERBLOCK"):
    for b in list(range(0, 8)) + list(range(30, 34)) + list(range(120, 124)) + list(range(280, 296)):
        if b < len(rel):
            print(b, " ".join(f"{rel[b, k]:6.2f}" for k in (0, 4, 5, 1)))
