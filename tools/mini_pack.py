import sys, os, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_jagged_paths as T
n = int(sys.argv[1]); ml = int(sys.argv[2])
lens, offs, plen = T._inputs(n, ml, seed=1)
pool = np.random.default_rng(2).integers(0, 256, plen * 8 + 8, dtype=np.uint8)
p, got, t = T._pack(lens, offs, pool, 8, [(0, 8)], 'i32', cap_extra=3)
pw, want, tw = T._expect(lens, offs, pool[:plen * 8], 8, [(0, 8)], 'i32')
print(n, ml, 'ok' if (t == tw and p.tobytes() == pw.tobytes() and got == want) else 'MISMATCH', t, tw, flush=True)
