"""Case-study kernel (K5) and the fused transfer + calibrate path vs the
reference's golden energies/noises (bit-exact: the reference pins energy bytes
across layouts, test_detector.py:200-214)."""

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, HOST, PINNED, aos_collection, to_host_planes
from oracle import restate as R
from paper_2511_04853_b200 import layouts as ly
from paper_2511_04853_b200 import memctx as mc
from paper_2511_04853_b200 import sensor, transfer as tr
from skhelp import golden

pytestmark = pytest.mark.gpu

EVENTS = ["sensor_16x16_s5.npz", "sensor_64x64_s3.npz", "sensor_101x37_s11.npz"]


@pytest.mark.parametrize("name", EVENTS)
def test_behaviors_on_device_match_reference(name):
    g = golden(name)
    n = int(g["w"] * g["h"])
    host = aos_collection(sensor.SENSOR_SCHEMA, g["aos"], n, HOST)
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    assert tr.copy_collection(dev, host) == "b200-convert"
    with mc.execution_scope(mc.CUDA):
        dev.funcs.calibrate_energy()
        noise = dev.funcs.get_noise()
        energy = dev.column("energy").read()
    assert energy.tobytes() == g["energy"].tobytes()
    assert noise.numpy().tobytes() == g["noise"].tobytes()


@pytest.mark.parametrize("name", EVENTS)
@pytest.mark.parametrize("src_ctx", ["host", "pinned", "cuda"])
def test_fused_transfer_calibrate_matches_reference(name, src_ctx):
    g = golden(name)
    n = int(g["w"] * g["h"])
    src = aos_collection(sensor.SENSOR_SCHEMA, g["aos"], n, PINNED if src_ctx == "pinned" else HOST)
    if src_ctx == "cuda":
        d = sk.Collection(sensor.SENSOR_SCHEMA, ly.AOS, CUDA)
        tr.copy_collection(d, src)
        src = d
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    noise = sensor.transfer_calibrate(dev, src)
    assert noise.numpy().tobytes() == g["noise"].tobytes()
    planes = to_host_planes(dev)
    assert planes["energy#0"] == g["energy"].tobytes()
    recs = g["aos"].view(R.SENSOR_AOS_DTYPE)
    assert planes["counts#0"] == np.ascontiguousarray(recs["counts"]).tobytes()
    assert planes["calibration_data.noise_B#0"] == np.ascontiguousarray(recs["calibration_data"]["noise_B"]).tobytes()


def test_golden_values_and_exact_doubling():
    # test_detector.py:184-187 and 228-239
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    host = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, HOST)
    host.resize(3)
    host.column("counts").np[:] = [100, 0, 7]
    host.column("calibration_data.parameter_A").np[:] = [0.5, 1.0, 1.25]
    host.column("calibration_data.parameter_B").np[:] = [2.0, 0.0, 0.75]
    host.column("calibration_data.noise_A").np[:] = [1.25, 1.0, 1.25]
    host.column("calibration_data.noise_B").np[:] = [0.75, 0.1, 0.75]
    host.column("calibration_data.noisy").np[:] = [False, False, True]
    tr.copy_collection(dev, host)
    sensor.calibrate_collection(dev)
    nz = sensor.noise_for_collection(dev).numpy()
    with mc.execution_scope(mc.CUDA):
        e = dev.column("energy").read()
    assert e[0] == np.float32(52.0) and e[1] == np.float32(0.0)
    assert nz[1] == np.float32(0.1)
    quiet = np.float32(1.25) * np.sqrt(e[2]) + np.float32(0.75)
    assert nz[2] == np.float32(2.0) * quiet


def test_batched_full_size_events_vs_oracle():
    """Config 2 shape: 436 x 436 = 190,096 cells per event, 8 events batched."""
    evs = [R.generate_event(436, 436, seed=s, density=0.002) for s in range(8)]
    recs = np.concatenate([R.sensor_aos(ev) for ev in evs])
    n = recs.size
    src = aos_collection(sensor.SENSOR_SCHEMA, recs, n, PINNED)
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    noise = sensor.transfer_calibrate(dev, src).numpy()
    e = R.calibrate(recs["counts"], recs["calibration_data"]["parameter_A"], recs["calibration_data"]["parameter_B"])
    nz = R.noise(e, recs["calibration_data"]["noise_A"], recs["calibration_data"]["noise_B"],
                 recs["calibration_data"]["noisy"])
    assert to_host_planes(dev)["energy#0"] == e.tobytes()
    assert noise.tobytes() == nz.tobytes()


def test_special_values_vs_oracle():
    rng = np.random.default_rng(11)
    n = 65537
    recs = np.zeros(n, R.SENSOR_AOS_DTYPE)
    recs["counts"] = rng.integers(0, np.iinfo(np.uint64).max, n, dtype=np.uint64, endpoint=True)
    cal = recs["calibration_data"]
    for k in ("parameter_A", "parameter_B", "noise_A", "noise_B"):
        cal[k] = (rng.standard_normal(n) * 10.0 ** rng.integers(-40, 30, n)).astype(np.float32)
    cal["parameter_A"][:16] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1e-45, -1e-45, 3e38] * 2
    cal["noisy"] = rng.integers(0, 2, n).astype(bool)
    src = aos_collection(sensor.SENSOR_SCHEMA, recs, n, HOST)
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    with np.errstate(all="ignore"):
        e = R.calibrate(recs["counts"], cal["parameter_A"], cal["parameter_B"])
        nz = R.noise(e, cal["noise_A"], cal["noise_B"], cal["noisy"])
    noise = sensor.transfer_calibrate(dev, src).numpy()
    assert to_host_planes(dev)["energy#0"] == e.tobytes()
    assert noise.tobytes() == nz.tobytes()


COLS = {"type": "type", "counts": "counts", "noisy": "calibration_data.noisy",
        "parameter_A": "calibration_data.parameter_A", "parameter_B": "calibration_data.parameter_B",
        "noise_A": "calibration_data.noise_A", "noise_B": "calibration_data.noise_B"}


@pytest.mark.parametrize("name", EVENTS)
def test_device_event_generation_matches_reference(name):
    """On-device splitmix64 events == the reference's generate_event columns."""
    g = golden(name)
    w, h = int(g["w"]), int(g["h"])
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(dev, w, h, [int(g["seed"])], float(g["density"]))
    planes = to_host_planes(dev)
    for ev_key, leaf in COLS.items():
        want = np.ascontiguousarray(g[f"ev:{ev_key}"])
        if want.dtype == np.bool_:
            want = want.view(np.uint8)
        assert planes[f"{leaf}#0"] == want.tobytes(), ev_key
    assert planes["energy#0"] == bytes(4 * w * h)


def test_batched_device_events_vs_oracle():
    seeds = [0, 1, 0xDEADBEEF, (1 << 64) - 1]
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(dev, 436, 436, seeds, 0.002)
    planes = to_host_planes(dev)
    evs = [R.generate_event(436, 436, s, 0.002) for s in seeds]
    for ev_key, leaf in COLS.items():
        want = np.concatenate([ev[ev_key] for ev in evs])
        assert planes[f"{leaf}#0"] == want.view(np.uint8).tobytes(), ev_key


def test_host_resident_collection_is_refused():
    host = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, HOST)
    with pytest.raises(sk.AccessError):
        host.funcs.calibrate_energy()


@pytest.mark.parametrize("ctx", ["host", "cuda"])
def test_fill_sensor_collection_and_object_behaviors(ctx):
    """fill_sensor_collection (reconstruct.py:142-154) on host and device collections, then the object-target
    behaviors (detector/schemas.py:15-26): host records run the reference's scalar arithmetic, device records
    run K5 over one record. Both equal the collection-level result."""
    ev = R.generate_event(101, 37, seed=11, density=0.01)
    info = mc.ContextInfo.host() if ctx == "host" else CUDA
    c = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, info)
    scope = mc.HOST if ctx == "host" else mc.CUDA
    with mc.execution_scope(scope):
        sensor.fill_sensor_collection(c, ev)
        assert c.size() == 101 * 37
        for i in (0, 17, 3736):
            c.record(i).funcs.calibrate_energy()
        energy = c.column("energy").read()
        noise_one = [c.record(i).funcs.get_noise() for i in (0, 17, 3736)]
    want_e = R.calibrate(ev["counts"], ev["parameter_A"], ev["parameter_B"])
    want_n = R.noise(want_e, ev["noise_A"], ev["noise_B"], ev["noisy"])
    for k, i in enumerate((0, 17, 3736)):
        assert energy[i].tobytes() == want_e[i].tobytes()
        assert np.float32(noise_one[k]).tobytes() == want_n[i].tobytes()
    assert not energy[1:17].any()  # only the records asked for were calibrated


def test_fused_option_through_copy_collection():
    """copy_collection(dst, src, {"fuse": "sensor_funcs"}) + funcs.calibrate_energy() + funcs.get_noise():
    the reference's prepare sequence in one HBM pass, same bytes as the separate path and the reference."""
    g = golden("sensor_64x64_s3.npz")
    n = int(g["w"] * g["h"])
    host = aos_collection(sensor.SENSOR_SCHEMA, g["aos"], n, PINNED)
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    assert tr.copy_collection(dev, host, {"fuse": "sensor_funcs"}) == "b200-convert"
    with mc.execution_scope(mc.CUDA):
        dev.funcs.calibrate_energy()
        noise = dev.funcs.get_noise()
        assert noise is dev.funcs.get_noise()  # the fused column, no second kernel
        energy = dev.column("energy").read()
    assert energy.tobytes() == g["energy"].tobytes()
    assert noise.numpy().tobytes() == g["noise"].tobytes()
    # a later plain transfer drops the fused marker: the behaviors run their kernels again
    tr.copy_collection(dev, host)
    with mc.execution_scope(mc.CUDA):
        assert not dev.column("energy").read().any()  # the AoS records carry energy 0
        dev.funcs.calibrate_energy()
        assert dev.column("energy").read().tobytes() == g["energy"].tobytes()
    with pytest.raises(sk.TransferError):
        tr.copy_collection(dev, host, {"fuse": "particle_funcs"})


def test_skev_files_into_a_device_collection(tmp_path):
    """SKEV event files (the reference's format, events.py:147-197) loaded straight into device planes, then
    the case-study kernel: same energies and noises as the oracle on the same events."""
    specs = [(64, 64, 3, 0.01), (64, 64, 4, 0.01)]
    host = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, HOST)
    paths = [tmp_path / f"{i}.skev" for i in range(2)]
    gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(gen, 64, 64, [3, 4], 0.01)
    tr.copy_collection(host, gen)
    sensor.save_events(host, paths, specs)
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    with mc.execution_scope(mc.CUDA):
        assert sensor.load_events(paths, dev) == specs
        dev.funcs.calibrate_energy()
        noise = dev.funcs.get_noise().numpy()
        energy = dev.column("energy").read()
    for i, seed in enumerate((3, 4)):
        ev = R.generate_event(64, 64, seed=seed, density=0.01)
        e = R.calibrate(ev["counts"], ev["parameter_A"], ev["parameter_B"])
        sl = slice(i * 4096, (i + 1) * 4096)
        assert energy[sl].tobytes() == e.tobytes()
        assert noise[sl].tobytes() == R.noise(e, ev["noise_A"], ev["noise_B"], ev["noisy"]).tobytes()
