"""The oracle restatement pinned against golden vectors from the real reference."""

import numpy as np
import pytest

from oracle import restate as R
from skhelp import golden

OBJ8_FIELDS = [(f"f{i}", "f32" if i % 2 == 0 else "i32", 1) for i in range(8)]
PARTICLE_FIELDS = [("energy", "f32", 1), ("x", "f32", 1), ("y", "f32", 1), ("origin", "u64", 1),
                   ("x_variance", "f32", 1), ("y_variance", "f32", 1), ("significance.value", "f32", 4),
                   ("E_contribution.value", "f32", 4), ("noisy_count.value", "u8", 4)]


def test_obj8_aos_to_planes_matches_reference():
    g = golden("obj8.npz")
    n = int(g["n"])
    recs = g["aos"].view(R.packed_dtype(OBJ8_FIELDS))
    planes = R.aos_to_planes(recs)
    for name, _, _ in OBJ8_FIELDS:
        assert planes[name][0].view(np.uint8).tobytes() == g[f"plane:{name}#0"].tobytes(), name
    back = R.planes_to_aos(planes, recs.dtype, n)
    assert back.tobytes() == g["aos"].tobytes()


def test_particle_multislot_planes_match_reference():
    g = golden("particle.npz")
    dt = R.packed_dtype(PARTICLE_FIELDS)
    assert dt.itemsize == int(g["stride"]) == 64  # test_layouts.py:234-241
    recs = g["aos"].view(dt)
    planes = R.aos_to_planes(recs)
    for name, _, ext in PARTICLE_FIELDS:
        for k in range(ext):
            assert planes[name][k].view(np.uint8).tobytes() == g[f"plane:{name}#{k}"].tobytes(), (name, k)


@pytest.mark.parametrize("name", ["sensor_16x16_s5.npz", "sensor_64x64_s3.npz", "sensor_101x37_s11.npz"])
def test_sensor_event_calibration_and_noise_match_reference(name):
    g = golden(name)
    ev = R.generate_event(int(g["w"]), int(g["h"]), int(g["seed"]), float(g["density"]))
    for k, v in ev.items():
        assert np.array_equal(v, g[f"ev:{k}"]), k
    aos = R.sensor_aos(ev)
    assert aos.tobytes() == g["aos"].tobytes()
    e = R.calibrate(ev["counts"], ev["parameter_A"], ev["parameter_B"])
    assert e.tobytes() == g["energy"].tobytes()
    nz = R.noise(e, ev["noise_A"], ev["noise_B"], ev["noisy"])
    assert nz.tobytes() == g["noise"].tobytes()


def test_calibration_golden_value():
    # test_detector.py:184-187: counts=100, A=0.5, B=2 -> 52.0; noise(0) = nB
    e = R.calibrate(np.array([100], np.uint64), np.float32([0.5]), np.float32([2.0]))
    assert e[0] == np.float32(52.0)
    nz = R.noise(np.float32([0.0]), np.float32([1.0]), np.float32([0.1]), np.array([False]))
    assert nz[0] == np.float32(0.1)


@pytest.mark.parametrize("label,dtype", [("i32", np.int32), ("u8", np.uint8), ("u16", np.uint16), ("i64", np.int64)])
def test_jagged_pack_matches_reference(label, dtype):
    g = golden("jagged.npz")
    lens = g[f"{label}:lens"]
    offsets = np.concatenate([[0], np.cumsum(lens.astype(np.int64))[:-1]])
    prefix, pool = R.jagged_pack(lens, offsets, g[f"{label}:pool_in"], dtype)
    assert prefix.dtype == g[f"{label}:prefix"].dtype
    assert prefix.tobytes() == g[f"{label}:prefix"].tobytes()
    assert pool.tobytes() == g[f"{label}:pool"].tobytes()


def test_jagged_u8_index_wraps_like_reference():
    g = golden("jagged.npz")
    assert int(g["u8:lens"].astype(np.int64).sum()) > 255  # the fixture exercises the wrap


def test_multi_leaf_members_match_import_external():
    g = golden("jagged.npz")
    lens = g["hits:lens"]
    offsets = np.concatenate([[0], np.cumsum(lens.astype(np.int64))[:-1]])
    p, adc = R.jagged_pack(lens, offsets, g["hits:adc_in"], np.int32)
    _, t = R.jagged_pack(lens, offsets, g["hits:t_in"], np.int32)
    assert p.tobytes() == g["hits:prefix"].tobytes()
    assert adc.tobytes() == g["hits:adc"].tobytes() and t.tobytes() == g["hits:t"].tobytes()


def test_splitmix_known_answers():
    g = golden("splitmix.npz")
    for seed in (0, 1, 0xDEADBEEF, (1 << 64) - 1):
        assert np.array_equal(R.mix_stream(seed, 0, 64), g[f"seed{seed}"])
        assert np.array_equal(R.mix_stream(seed, 17, 10), g[f"seed{seed}_off17"])


def test_aosoa_restatement_layout():
    recs = np.zeros(5, R.packed_dtype([("a", "f64", 1), ("b", "i32", 1)]))
    recs["a"] = [1.5, -2.0, np.nan, 1e39, 3.0]
    recs["b"] = [1, 2, 3, 4, 5]
    img = np.frombuffer(R.to_aosoa(recs, [("b", "i32"), ("a", "f32")], 4), np.uint8)
    assert img.size == 2 * 32  # 2 tiles x (4*4 + 4*4) bytes
    t0 = img[:32]
    assert np.array_equal(t0[:16].view(np.int32), [1, 2, 3, 4])
    assert t0[16:].view(np.float32)[0] == np.float32(1.5)
    t1 = img[32:]
    assert np.array_equal(t1[:16].view(np.int32), [5, 0, 0, 0])  # tail lanes zero


@pytest.mark.parametrize("name", ["particles_16x16_s5.npz", "particles_64x64_s3.npz", "particles_101x37_s11.npz",
                                  "particles_160x120_s21.npz"])
def test_reconstruction_restatement_matches_reference(name):
    g = golden(name)
    w, h = int(g["w"]), int(g["h"])
    ev = R.generate_event(w, h, int(g["seed"]), float(g["density"]))
    e = R.calibrate(ev["counts"], ev["parameter_A"], ev["parameter_B"])
    nz = R.noise(e, ev["noise_A"], ev["noise_B"], ev["noisy"])
    got = R.reconstruct(e, nz, ev["type"], ev["noisy"], w, h)
    for k in ("energy", "x", "y", "origin", "x_variance", "y_variance", "significance", "E_contribution",
              "noisy_count", "sensor_lens", "sensors"):
        assert got[k].tobytes() == g[k].tobytes(), k
