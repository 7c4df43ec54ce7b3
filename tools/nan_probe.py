import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat, layouts as ly, sensor, memctx as mc, transfer as tr
from paper_2511_04853_b200.devarray import DeviceArray
from gpuhelp import aos_collection, HOST, CUDA, to_host_planes
from oracle import restate as R
n = 16
recs = np.zeros(n, R.SENSOR_AOS_DTYPE)
recs["counts"] = 3
cal = recs["calibration_data"]
cal["parameter_A"] = np.nan; cal["parameter_B"] = 1.0; cal["noise_A"] = 2.0; cal["noise_B"] = 0.5
cal["noisy"] = [True, False] * 8
for ctx in ("host", "cuda"):
    src = aos_collection(sensor.SENSOR_SCHEMA, recs, n, HOST)
    if ctx == "cuda":
        d = sk.Collection(sensor.SENSOR_SCHEMA, ly.AOS, CUDA); tr.copy_collection(d, src); src = d
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    nz = sensor.transfer_calibrate(dev, src).numpy()
    print(ctx, "fused noise", [hex(x) for x in nz.view(np.uint32)[:4]])
    nz2 = sensor.noise_for_collection(dev).numpy()
    print(ctx, "standalone noise", [hex(x) for x in nz2.view(np.uint32)[:4]])
with np.errstate(all="ignore"):
    e = R.calibrate(recs["counts"], cal["parameter_A"], cal["parameter_B"])
    print("oracle", [hex(x) for x in R.noise(e, cal["noise_A"], cal["noise_B"], cal["noisy"]).view(np.uint32)[:4]])
