"""Tiling sweep for the conversion engine (run on a B200 via gpurun).

Prints one JSON line per (workload, setting) with the device GB/s over the
algorithmic bytes, plus live copy references (cudaMemcpy D2D and torch copy_)
measured in the same process.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, convert as cv, layouts as ly, memctx as mc  # noqa: E402
from paper_2511_04853_b200 import schema as sc, sensor, transfer as tr, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

DEV = 0
CUDA = mc.ContextInfo.cuda(DEV)


def coll(schema, kind, n):
    c = sk.Collection(schema, kind, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    return c


def timed(fn, steps=10, warmup=3):
    for _ in range(warmup):
        fn()
    nat.sync(DEV)
    a, b = nat.Event(), nat.Event()
    a.record(DEV)
    for _ in range(steps):
        fn()
    b.record(DEV)
    return a.elapsed_ms(b) / steps


def live_copy_refs(nbytes):
    x = DeviceArray(nbytes, np.uint8, CUDA)
    y = DeviceArray(nbytes, np.uint8, CUDA)
    ms = timed(lambda: nat.memcpy(y.ptr, x.ptr, nbytes, DEV))
    out = {"memcpy_d2d_gbs": round(2 * nbytes / ms / 1e6, 1)}
    x.free()
    y.free()
    a = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        b.copy_(a)
    e.record()
    torch.cuda.synchronize()
    out["torch_copy_gbs"] = round(2 * nbytes / (s.elapsed_time(e) / 10) / 1e6, 1)
    return out


SETTINGS = [dict()] + [dict(SK_TILE_BYTES=str(t), SK_CTAS=str(c), SK_STAGES=str(s))
                        for t in (8192, 12288, 16384, 24576, 32768) for c in (2, 3, 4, 6) for s in (2, 3)]
if os.environ.get("SWEEP_SHORT"):
    SETTINGS = [dict()]
if os.environ.get("SWEEP_BIG"):
    SETTINGS = [dict()] + [dict(SK_TILE_BYTES=str(t), SK_CTAS=str(c), SK_STAGES="2")
                           for t in (32768, 40960, 49152, 65536) for c in (1, 2)]


def main():
    which = sys.argv[1:] or ["obj8", "obj8_p2a", "sensor", "track"]
    print(json.dumps({"live": live_copy_refs(3_200_000_000)}), flush=True)
    n = 100_000_000
    jobs = {}
    if "obj8" in which or "obj8_p2a" in which:
        a = coll(wl.OBJ8_SCHEMA, ly.AOS, n)
        p = coll(wl.OBJ8_SCHEMA, ly.PER_FIELD, n)
        wl.fill_random_device(a.layout._struct_buf.ptr, n * 32, 1, DEV)
        if "obj8" in which:
            jobs["obj8_a2p"] = (lambda: tr.copy_collection(p, a, {"async": True}), n * 64)
        if "obj8_p2a" in which:
            jobs["obj8_p2a"] = (lambda: tr.copy_collection(a, p, {"async": True}), n * 64)
    if "sensor" in which:
        cells = 64 * 436 * 436
        sa = coll(sensor.SENSOR_SCHEMA, ly.AOS, cells)
        sp = coll(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cells)
        wl.fill_random_device(sa.layout._struct_buf.ptr, cells * 30 // 8 * 8, 2, DEV)
        noise = DeviceArray(cells, np.float32, CUDA)
        jobs["sensor_fused"] = (lambda: sensor.transfer_calibrate(sp, sa, noise, sync=False), cells * 64)
        jobs["sensor_a2p"] = (lambda: tr.copy_collection(sp, sa, {"async": True}), cells * 60)
    if "track" in which:
        ta = coll(wl.TRACK_SCHEMA, ly.AOS, n)
        wl.fill_random_device(ta.layout._struct_buf.ptr, n * 60, 4, DEV)
        fields = [sk.AosoaField("pz", "f32"), sk.AosoaField("px", "f32"), sk.AosoaField("x", "f32"),
                  sk.AosoaField("charge", "i32")]
        ao = sk.Aosoa(n, 128, fields, CUDA)
        jobs["track_aosoa"] = (lambda: sk.to_aosoa(ta, fields, 128, out=ao, sync=False), n * 76)
    for name, (fn, nbytes) in jobs.items():
        for st in SETTINGS:
            for k in ("SK_TILE_BYTES", "SK_STAGES", "SK_CTAS", "SK_CACHE_HINT"):
                os.environ.pop(k, None)
            os.environ.update(st)
            ms = timed(fn)
            print(json.dumps({"job": name, "setting": st, "ms": round(ms, 4), "gbs": round(nbytes / ms / 1e6, 1)}),
                  flush=True)


if __name__ == "__main__":
    main()
