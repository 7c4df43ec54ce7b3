"""Small invocations of every kernel family for compute-sanitizer runs
(memcheck / racecheck / synccheck): jagged scan + both gathers + scatter,
conversion word/element/specialised paths, sensor fused, reco."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_jagged_paths as J  # noqa: E402

lens, offs, plen = J._inputs(3000, 20, seed=1)
pool = np.random.default_rng(1).integers(0, 256, plen * 8 + 8, dtype=np.uint8)
J._pack(lens, offs, pool, 8, [(0, 8)], "i32", cap_extra=99)            # async gather
J._pack(lens, offs, pool, 8, [(0, 8)], "i32", dst_shift=8)             # register gather
pool15 = np.random.default_rng(2).integers(0, 256, plen * 15, dtype=np.uint8)
J._pack(lens, offs, pool15, 15, [(0, 4), (4, 8), (12, 2), (14, 1)], "i64")  # generic table
lens2, offs2, plen2 = J._inputs(2000, 60, seed=3)
pool2 = np.random.default_rng(3).integers(0, 256, plen2 * 8, dtype=np.uint8)
J._pack(lens2, offs2, pool2, 8, [(0, 8)], "u16")                       # wrapping prefix
J._pack(lens2, offs2, pool2, 8, [(0, 4)], "i32", cap_extra=10)         # 4-byte async
J._pack(lens2, offs2, pool2, 8, [(0, 8)], "i32", cap_extra=-100)       # overflow: gathers nothing
lens3 = np.random.default_rng(4).integers(0, 4, 5000).astype(np.int32)
lens3[100:200] = 1000                                                   # a sub-tile over the queueing threshold
order = np.random.default_rng(5).permutation(lens3.size)
gaps = lens3[order].astype(np.int64) + 1
offs3 = np.empty(lens3.size, np.int64)
offs3[order] = np.concatenate([[0], np.cumsum(gaps)[:-1]])
pool3 = np.random.default_rng(6).integers(0, 256, int(gaps.sum()) * 8, dtype=np.uint8)
J._pack(lens3, offs3, pool3, 8, [(0, 8)], "i64")                       # fused: queued sub-tile shared out
J._pack(lens2, offs2, pool2, 8, [(0, 8)], "i32", lens_shift=1, prefix_shift=1)  # scalar block sums / prefix
J._pack(lens2, offs2, pool2, 8, [(0, 4), (4, 4)], "i32")               # fused, record staged + split drain
pool16 = np.random.default_rng(7).integers(0, 256, plen2 * 16, dtype=np.uint8)
J._pack(lens2, offs2, pool16, 16, [(8, 8), (0, 4)], "i64")             # 16-byte records
J.test_scatter_over_given_prefix.__wrapped__ if hasattr(J.test_scatter_over_given_prefix, "__wrapped__") else None

import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import layouts as ly, memctx as mc, sensor, transfer as tr, workloads as wl  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)
for n in (1, 5000, 70001):
    recs = wl.obj8_records(n, seed=n)
    h = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.pinned())
    h.resize(n)
    h.layout._struct_buf._data[: n * 32] = recs.view(np.uint8)
    d = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(d, h)
    back = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, CUDA)
    tr.copy_collection(back, d)
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
sensor.generate_events(gen, 40, 30, range(2), 0.01)
a = sk.Collection(sensor.SENSOR_SCHEMA, ly.AOS, CUDA)
tr.copy_collection(a, gen)
p = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402
noise = DeviceArray(len(a), np.float32, CUDA)
sensor.transfer_calibrate(p, a, noise)
parts = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, CUDA)
sensor.reconstruct_from_collection(p, 40, 30, out=parts, events=2, noise=noise)
# the scalar tile pass (w % 4 != 0) on dense, tied events: long blocker chains, several rounds, and more
# particles than the output's first guess (the grow-and-write-again path)
rng = np.random.default_rng(5)
dw, dh, dev_n = 37, 23, 3
recs = np.zeros(dw * dh * dev_n, sensor.SENSOR_AOS_DTYPE)
recs["energy"] = np.array([1.0, 3.0, 6.0, 7.0, 8.0, 50.0], np.float32)[rng.integers(0, 6, recs.size)]
recs["type"] = rng.integers(0, 4, recs.size)
dense_h = sk.Collection(sensor.SENSOR_SCHEMA, ly.AOS, mc.ContextInfo.pinned())
dense_h.resize(recs.size)
dense_h.layout._struct_buf._data[: recs.nbytes] = recs.view(np.uint8)
dense = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
tr.copy_collection(dense, dense_h)
ones = DeviceArray.from_numpy(np.ones(recs.size, np.float32), CUDA)
sensor.reconstruct_from_collection(dense, dw, dh, events=dev_n, noise=ones)
# AoSoA: AoS -> AoSoA (record groups), per_field -> AoSoA and AoSoA -> per_field (block transform),
# AoSoA -> AoS (record groups reading AoSoA blocks)
for m in (3, 1001):
    trk = sk.Collection(wl.TRACK_SCHEMA, ly.AOS, mc.ContextInfo.pinned())
    trk.resize(m)
    trk.layout._struct_buf._data[: m * 60] = wl.track_records(m).view(np.uint8)
    ta = sk.Collection(wl.TRACK_SCHEMA, ly.AOS, CUDA)
    tr.copy_collection(ta, trk)
    tp = sk.Collection(wl.TRACK_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(tp, ta)
    flds = [sk.AosoaField("pz", "f32"), sk.AosoaField("charge", "i32"), sk.AosoaField("id", "u64")]
    for src in (ta, tp):
        ao = sk.to_aosoa(src, flds, 32)
        sk.from_aosoa(ao, tp)
        sk.from_aosoa(ao, ta)
        ao.free()
# round 2: segment validation (fused and validate + scan + gather), batched device splices, K5 alone with
# ragged tails, the device compare
J._pack_raw(np.array([3, -1, 2, 0], np.int32), np.array([0, 0, 100, 1 << 40], np.int64), 5, [(0, 8)])
J._pack_raw(np.array([3, 1, 2], np.int32), np.array([0, 4, 9], np.int64), 8, [(2, 2)], fused=False)
with mc.execution_scope(mc.CUDA):
    parts.insert_records(3, 5)
    parts.erase_records(1, 4)
    parts.resize(len(parts) + 37)
    sensor.calibrate_collection(p)
    sensor.noise_for_collection(p, noise)
for m in (1, 7, 4099):
    c = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(c, m, 1, range(1), 0.0)
    sensor.calibrate_collection(c)
    sensor.noise_for_collection(c)
import ctypes  # noqa: E402
from paper_2511_04853_b200 import _native as nat  # noqa: E402
cnt = DeviceArray(1, np.uint64, CUDA)
nat.call("sk_compare_bytes", a.layout._struct_buf.ptr, a.layout._struct_buf.ptr + 3, 1001, cnt.ptr, nat.stream(0))
nat.sync(0)
# first fill of a fresh device collection: the prefix-only pack (capacity 0), grow, then the register
# scatter over the prefix, with a skewed record (queued group)
from paper_2511_04853_b200 import jagged as _jg  # noqa: E402

_fl = np.random.default_rng(11).integers(0, 6, 3000).astype(np.int32)
_fl[700] = 9000
_fo, _fp = J._tiled_inputs(_fl, seed=12)
_fc = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(0))
with mc.execution_scope(mc.CUDA):
    _fc.resize(_fl.size)
_jg.pack(_fc, "members", _fl, _fo, np.random.default_rng(13).integers(0, 2**63, _fp, dtype=np.uint64))
print("sanitize paths done", len(parts))
