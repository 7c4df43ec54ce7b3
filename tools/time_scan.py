"""Device time of the jagged scan / gather / fused pack on config 3 (1M clusters).

Launches are queued behind a ~2 ms device fill so the GPU never waits on the
host: the event pair then brackets GPU time only."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_04853_b200 import _native as nat, memctx as mc, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
n = int(os.environ.get("N", 1_000_000))
HITS = bool(os.environ.get("HITS"))  # variant 3b: {adc i32, t f32} members into two pools
lens, offsets, pool = wl.cluster_inputs(n, seed=7, member_dtype=wl.HIT_DTYPE if HITS else np.uint64)
if HITS:
    pool = pool.view(np.uint8)
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
total = DeviceArray(2, np.int64, CUDA)
out = DeviceArray(cap, np.uint64, CUDA)
out2 = DeviceArray(cap, np.uint32, CUDA)
s = nat.stream(0)
big = DeviceArray(12 << 30, np.uint8, CUDA)
I32 = nat.TYPE_CODES["i32"]
NF = 2 if HITS else 1
foff = (C.c_int64 * NF)(*([0, 4] if HITS else [0]))
fsz = (C.c_int32 * NF)(*([4, 4] if HITS else [8]))
dst = (C.c_void_p * NF)(*([out.ptr, out2.ptr] if HITS else [out.ptr]))


def scan():
    nat.call("sk_jagged_scan", n, d_lens.ptr, I32, prefix.ptr, I32, scratch.ptr, scratch.n, total.ptr, s)


def scatter():
    nat.call("sk_jagged_scatter", n, prefix.ptr, I32, d_off.ptr, d_pool.ptr, 8, NF, foff, fsz, dst, T, s)


def pack():
    nat.call("sk_jagged_pack", n, d_lens.ptr, I32, prefix.ptr, I32, d_off.ptr, d_pool.ptr, d_pool.nbytes // 8, 8, NF,
             foff, fsz, dst,
             cap, scratch.ptr, scratch.n, total.ptr, s)


def device_us(fn, reps=40):
    for _ in range(3):
        fn()
    nat.sync(0)
    a, b = nat.Event(), nat.Event()
    nat.call("sk_fill_random", big.ptr, big.n, 1, 0, s)  # keeps the GPU busy while the host queues
    a.record(0)
    for _ in range(reps):
        fn()
    b.record(0)
    nat.sync(0)
    return a.elapsed_ms(b) / reps * 1e3


def memcpy4():
    nat.memcpy(out.ptr, d_lens.ptr, n * 4, 0)


res = {"scan_us": device_us(scan), "pack_us": device_us(pack), "memcpy_4MB_us": device_us(memcpy4)}
scan()
res["scatter_us"] = device_us(scatter)
nat.sync(0)
assert (prefix.numpy()[1:].astype(np.int64) == np.cumsum(lens)).all()
algo = n * 16 + T * 16
res["pack_gbs"] = round(algo / res["pack_us"] / 1e3, 1)
print({k: round(v, 1) for k, v in res.items()})

if os.environ.get("FLOORS"):
    small = DeviceArray(1 << 12, np.int32, CUDA)
    sp = DeviceArray(1 << 12 + 1, np.int32, CUDA)

    def scan_small():
        nat.call("sk_jagged_scan", 1000, small.ptr, I32, sp.ptr, I32, scratch.ptr, scratch.n, total.ptr, s)

    print({"memset_4B_us": round(device_us(lambda: nat.memset(out.ptr, 0, 4, 0)), 2),
           "memset_4MB_us": round(device_us(lambda: nat.memset(out.ptr, 0, 4 << 20, 0)), 2),
           "scan_n1000_us": round(device_us(scan_small), 2),
           "fill_4MB_us": round(device_us(lambda: nat.call("sk_fill_random", out.ptr, 4 << 20, 1, 0, s)), 2)})
