"""Config 2's prepare phase through soakit itself (baseline/_ref) with the plugin:
copy_collection(per_field@cuda, aos@pinned), funcs.calibrate_energy(),
funcs.get_noise() -- each step timed on its own (wall, synchronous)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_04853_b200 as sk  # noqa: E402
from oracle import cpu_baseline  # noqa: E402
from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, sensor  # noqa: E402

soakit = cpu_baseline.import_reference()
from paper_2511_04853_b200 import soakit_plugin  # noqa: E402

soakit_plugin.install()
from soakit.detector import schemas as ds  # noqa: E402

cells = 64 * 436 * 436
from paper_2511_04853_b200 import transfer as tr  # noqa: E402

gen_p = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(0))
sensor.generate_events(gen_p, 436, 436, range(64), 0.002, sync=True)
gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.AOS, mc.ContextInfo.cuda(0))
tr.copy_collection(gen, gen_p)
host = soakit.Collection(ds.SENSOR_SCHEMA, "aos", soakit_plugin.pinned_info())
host.resize(cells)
nat.memcpy(host.layout._struct_buf._data.ctypes.data, gen.layout._struct_buf.ptr, cells * 30, 0)
nat.sync(0)
devc = soakit.Collection(ds.SENSOR_SCHEMA, "per_field", soakit_plugin.cuda_info(0))


def t(fn, reps=5):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    nat.sync(0)
    return (time.perf_counter() - t0) / reps * 1e3


def cal():
    with soakit.memctx.execution_scope("cuda"):
        devc.funcs.calibrate_energy()


def noise():
    with soakit.memctx.execution_scope("cuda"):
        return devc.funcs.get_noise()


res = {"copy_collection_ms": t(lambda: (soakit.transfer.copy_collection(devc, host), nat.sync(0))),
       "calibrate_ms": t(cal), "get_noise_ms": t(noise),
       "np_empty_touch_49MB_ms": t(lambda: np.ones(cells, np.float32))}
res["prepare_ms"] = t(lambda: (soakit.transfer.copy_collection(devc, host), cal(), noise()))
print({k: round(v, 3) for k, v in res.items()})
