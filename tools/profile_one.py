"""Run one conversion job a few times (for ncu captures): python tools/profile_one.py JOB [reps]

JOB in: obj8_a2p obj8_p2a obj8_1m sensor_fused sensor_a2p sensor_calnoise track_aosoa particle_a2p jagged
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2511_04853_b200 as sk  # noqa: E402
from paper_2511_04853_b200 import _native as nat, jagged, layouts as ly, memctx as mc  # noqa: E402
from paper_2511_04853_b200 import schema as sc, sensor, transfer as tr, workloads as wl  # noqa: E402
from paper_2511_04853_b200.devarray import DeviceArray  # noqa: E402

CUDA = mc.ContextInfo.cuda(0)


def coll(schema, kind, n):
    c = sk.Collection(schema, kind, CUDA)
    with mc.execution_scope(mc.CUDA):
        c.reserve(n)
    with c.layout.engine_ops():
        c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
    return c


def job(name):
    n = 100_000_000
    if name.startswith("obj8"):
        n = 1_000_000 if name == "obj8_1m" else n  # config 1
        a, p = coll(wl.OBJ8_SCHEMA, ly.AOS, n), coll(wl.OBJ8_SCHEMA, ly.PER_FIELD, n)
        wl.fill_random_device(a.layout._struct_buf.ptr, n * 32, 1, 0)
        return (lambda: tr.copy_collection(p, a, {"async": True})) if name != "obj8_p2a" else \
            (lambda: tr.copy_collection(a, p, {"async": True}))
    if name.startswith("sensor"):
        cells = 64 * 436 * 436
        # real events (as bench.py config 2): random record bits would send the case-study
        # arithmetic through its NaN/denormal paths
        gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
        sensor.generate_events(gen, 436, 436, range(64), 0.002)
        a, p = coll(sensor.SENSOR_SCHEMA, ly.AOS, cells), coll(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cells)
        tr.copy_collection(a, gen)
        gen.free()
        noise = DeviceArray(cells, np.float32, CUDA)
        if name == "sensor_fused":
            return lambda: sensor.transfer_calibrate(p, a, noise, sync=False)
        if name == "sensor_calnoise":  # the standalone K5 kernels the drop-in behaviors launch
            tr.copy_collection(p, a)
            return lambda: (sensor.calibrate_collection(p, sync=False), sensor.noise_for_collection(p, noise, sync=False))
        return lambda: tr.copy_collection(p, a, {"async": True})
    if name == "particle_a2p":
        m = 50_000_000
        a, p = coll(sensor.PARTICLE_SCHEMA, ly.AOS, m), coll(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, m)
        wl.fill_random_device(a.layout._struct_buf.ptr, m * 64, 3, 0)
        return lambda: tr.copy_collection(p, a, {"async": True})
    if name == "track_aosoa":
        a = coll(wl.TRACK_SCHEMA, ly.AOS, n)
        wl.fill_random_device(a.layout._struct_buf.ptr, n * 60, 4, 0)
        fields = [sk.AosoaField("pz", "f32"), sk.AosoaField("px", "f32"), sk.AosoaField("x", "f32"),
                  sk.AosoaField("charge", "i32")]
        ao = sk.Aosoa(n, 128, fields, CUDA)
        return lambda: sk.to_aosoa(a, fields, 128, out=ao, sync=False)
    if name == "jagged":
        lens, offsets, pool = wl.cluster_inputs(1_000_000, seed=7)
        d = [DeviceArray.from_numpy(x, CUDA) for x in (lens, offsets, pool)]
        c = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, CUDA)
        with mc.execution_scope(mc.CUDA):
            c.resize(1_000_000)
        return lambda: jagged.pack(c, "members", *d)
    raise SystemExit(f"unknown job {name}")


if __name__ == "__main__":
    fn = job(sys.argv[1])
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
        fn()
    nat.sync(0)
