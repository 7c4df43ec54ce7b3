import os, sys, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2511_04853_b200 import _native as nat, memctx as mc
from paper_2511_04853_b200.devarray import DeviceArray
CUDA = mc.ContextInfo.cuda(0)
I32 = nat.TYPE_CODES["i32"]
small = DeviceArray.from_numpy(np.arange(4096, dtype=np.int32) % 7, CUDA)
sp = DeviceArray(4097, np.int32, CUDA)
scratch = DeviceArray(1 << 20, np.uint8, CUDA)
total = DeviceArray(1, np.int64, CUDA)
for _ in range(10):
    nat.call("sk_jagged_scan", 1000, small.ptr, I32, sp.ptr, I32, scratch.ptr, scratch.n, total.ptr, nat.stream(0))
nat.sync(0)
