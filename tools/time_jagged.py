"""Device time of sk_jagged_pack (config 3) queued behind a device fill, CUDA events.
usage: [SK_L2PRE=..] python tools/time_jagged.py [clusters ...]   (default 1M and 10M)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2511_04853_b200 import _native as nat, memctx as mc, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
PEAK = 6546.9
busy = DeviceArray(6 << 30, np.uint8, CUDA)
for n in [int(x) for x in sys.argv[1:]] or [1_000_000, 10_000_000]:
    lens, offs, pool = wl.cluster_inputs(n, seed=7)
    T = int(lens.sum())
    d = [DeviceArray.from_numpy(x, CUDA) for x in (lens, offs, pool)]
    prefix = DeviceArray(n + 1, np.int32, CUDA)
    out = DeviceArray(T + 4096, np.uint64, CUDA)
    need = C.c_size_t(0)
    nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
    scratch = DeviceArray(need.value, np.uint8, CUDA)
    total = DeviceArray(2, np.int64, CUDA)
    foff, fsz, dst = (C.c_int64 * 1)(0), (C.c_int32 * 1)(8), (C.c_void_p * 1)(out.ptr)
    s = nat.stream(0)

    def pack():
        nat.call("sk_jagged_pack", n, d[0].ptr, nat.TYPE_CODES["i32"], prefix.ptr, nat.TYPE_CODES["i32"], d[1].ptr,
                 d[2].ptr, pool.size, 8, 1, foff, fsz, dst, T + 4096, scratch.ptr, scratch.n, total.ptr, s)

    for _ in range(3):
        pack()
    nat.sync(0)
    steps = 20
    a, b = nat.Event(), nat.Event()
    nat.call("sk_fill_random", busy.ptr, busy.n, 1, 0, s)
    a.record(0)
    for _ in range(steps):
        pack()
    b.record(0)
    nat.sync(0)
    us = a.elapsed_ms(b) / steps * 1e3
    algo = n * 16 + T * 16
    ok = prefix.numpy()[-1] == np.int32(T) and int(total.numpy()[0]) == T
    print(f"clusters={n} members={T} pool_MB={pool.nbytes / 1e6:.0f} L2PRE={os.environ.get('SK_L2PRE', '0')} "
          f"us={us:.1f} gbs={algo / us / 1e3:.0f} frac={algo / us / 1e3 / PEAK:.3f} ok={ok}", flush=True)
    for x in (*d, prefix, out, scratch, total):
        x.free()
