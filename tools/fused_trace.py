"""Block timeline of the fused jagged pack (config 3) for the first 8 CTAs:
sub-tile sums, look-back, first table ready, block end (microseconds)."""
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
if os.environ.get("INORDER"):  # same lengths, segments packed in record order (sequential source reads)
    offsets = np.concatenate([[0], np.cumsum(lens.astype(np.int64))[:-1]])
T = int(lens.sum())
d_lens, d_off, d_pool = (DeviceArray.from_numpy(x, CUDA) for x in (lens, offsets, pool))
prefix = DeviceArray(n + 1, np.int32, CUDA)
need = C.c_size_t(0)
nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
cap = T + 1000
sbytes = -(-need.value // 256) * 256 + ((cap + 255) // 256 + 1) * 8
scratch = DeviceArray(sbytes, np.uint8, CUDA)
total = DeviceArray(1, np.int64, CUDA)
out = DeviceArray(cap, np.uint64, CUDA)
s = nat.stream(0)
big = DeviceArray(12 << 30, np.uint8, CUDA)
I32 = nat.TYPE_CODES["i32"]
foff = (C.c_int64 * 1)(0)
fsz = (C.c_int32 * 1)(8)
dst = (C.c_void_p * 1)(out.ptr)




def pack():
    nat.call("sk_jagged_pack", n, d_lens.ptr, I32, prefix.ptr, I32, d_off.ptr, d_pool.ptr, 8, 1, foff, fsz, dst,
             cap, scratch.ptr, scratch.n, total.ptr, s)


for _ in range(5):
    pack()
nat.sync(0)
buf = np.zeros(8 * 16 * 8, np.uint64)
nat.call("sk_jagged_pack", n, d_lens.ptr, I32, prefix.ptr, I32, d_off.ptr, d_pool.ptr, 8, 1, foff, fsz, dst,
         cap, scratch.ptr, scratch.n, total.ptr, s)
nat.call("sk_jagged_trace", buf.ctypes.data, buf.nbytes)
t = buf.reshape(8, 16, 8).astype(np.int64)
t0 = t[:, 0, 0][t[:, 0, 0] > 0].min()
for cta in range(8):
    w0, w1 = t[cta, 0], t[cta, 1]
    us = lambda a, b: (a - b) / 1e3 if a and b else float("nan")
    print(f"cta {cta}: start {us(w0[0], t0):6.2f}  sums {us(w0[1], w0[0]):5.2f}  lookback {us(w0[2], w0[1]):5.2f}  "
          f"first sub-tile ready (w0/w1) {us(w0[3], w0[2]):5.2f} / {us(w1[4], w0[2]):5.2f}  "
          f"block end (w0/w1) {us(w0[5], t0):6.2f} / {us(w1[6], t0):6.2f} us")

print("table-warp sub-tile detail (us): issue, load wait, tables, E wait, prefix, handover")
for cta in range(4):
    for w in range(2):
        for row in range(2):
            r = t[cta, 2 + 2 * w + row]
            if not r[0]:
                continue
            d = [(r[k + 1] - r[k]) / 1e3 if r[k + 1] and r[k] else float("nan") for k in range(6)]
            print(f"cta {cta} tw {w} sub {2 * row + w}: start {(r[0] - t0) / 1e3:6.2f} " +
                  " ".join(f"{v:5.2f}" for v in d))
if os.environ.get("RAW"):
    for row in range(6):
        print(row, [(int(v) - int(t0)) / 1e3 if v else 0 for v in t[0, row]])
