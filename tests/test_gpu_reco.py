"""Particle reconstruction on the GPU vs the reference's reconstruct_arrays
(golden particles, including a dense event with heavily overlapping deposit
windows) and vs the oracle on batched full-size events."""

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, HOST, aos_collection, to_host_planes
from oracle import restate as R
from paper_2511_04853_b200 import layouts as ly, memctx as mc, sensor, transfer as tr
from skhelp import golden

pytestmark = pytest.mark.gpu


FIELDS = ("energy", "x", "y", "origin", "x_variance", "y_variance")
ARRAYS = ("significance", "E_contribution", "noisy_count")


def _host_particles(coll):
    h = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, HOST)
    tr.copy_collection(h, coll)
    out = {k: np.array(h.column(k).read()) for k in FIELDS}
    for k in ARRAYS:
        out[k] = np.ascontiguousarray(np.array(h.column(k).read()).T)
    p = h.prefix_sums("sensors")
    out["sensor_lens"] = np.diff(p.astype(np.int64)).astype(np.int32)
    out["sensors"] = np.array(h.column("sensors").read())
    return out


def _compare(got, want, tag):
    for k in FIELDS + ARRAYS + ("sensor_lens", "sensors"):
        assert np.asarray(got[k]).tobytes() == np.asarray(want[k]).tobytes(), (tag, k)


@pytest.mark.parametrize("name", ["particles_16x16_s5.npz", "particles_64x64_s3.npz", "particles_101x37_s11.npz",
                                  "particles_160x120_s21.npz"])
def test_reconstruction_matches_reference(name):
    g = golden(name)
    w, h = int(g["w"]), int(g["h"])
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(dev, w, h, [int(g["seed"])], float(g["density"]))
    with mc.execution_scope(mc.CUDA):
        dev.funcs.calibrate_energy()
    parts = sensor.reconstruct_from_collection(dev, w, h)
    assert len(parts) == g["energy"].size and parts.event_counts == [g["energy"].size]
    _compare(_host_particles(parts), g, name)


def test_batched_full_size_events_vs_oracle():
    seeds, w, h = [0, 7, 0xDEADBEEF], 436, 436
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(dev, w, h, seeds, 0.002)
    with mc.execution_scope(mc.CUDA):
        dev.funcs.calibrate_energy()
        e = dev.column("energy").read()
    noise = sensor.noise_for_collection(dev).numpy()
    planes = to_host_planes(dev)
    typ = np.frombuffer(planes["type#0"], np.uint8)
    noisy = np.frombuffer(planes["calibration_data.noisy#0"], np.uint8).astype(bool)
    parts = sensor.reconstruct_from_collection(dev, w, h, events=len(seeds))
    got = _host_particles(parts)
    n = w * h
    lo = 0
    for i, _ in enumerate(seeds):
        want = R.reconstruct(e[i * n:(i + 1) * n], noise[i * n:(i + 1) * n], typ[i * n:(i + 1) * n],
                             noisy[i * n:(i + 1) * n], w, h)
        m = parts.event_counts[i]
        assert m == want["energy"].size
        sl = {k: got[k][lo:lo + m] for k in FIELDS + ARRAYS + ("sensor_lens",)}
        starts = np.concatenate([[0], np.cumsum(got["sensor_lens"].astype(np.int64))])
        sl["sensors"] = got["sensors"][starts[lo]:starts[lo + m]]
        _compare(sl, want, i)
        lo += m


def test_event_without_deposits_has_no_particles():
    dev = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(dev, 32, 32, [3], 0.0)
    with mc.execution_scope(mc.CUDA):
        dev.funcs.calibrate_energy()
    parts = sensor.reconstruct_from_collection(dev, 32, 32)
    assert len(parts) == 0 and parts.jagged_size("sensors") == 0


@pytest.mark.parametrize("name", ["particles_64x64_s3.npz", "particles_160x120_s21.npz"])
def test_export_particles_matches_reference_struct(name):
    """export_particles_from_collection (detector/baselines.py:104-120): the GPU reconstruction's particles as
    the reference's packed PARTICLE_AOS_DTYPE records + per-particle sensor lists, through K2 and one D2H."""
    g = golden(name)
    w, h = int(g["w"]), int(g["h"])
    ev = R.generate_event(w, h, seed=int(g["seed"]), density=float(g["density"]))
    cells = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(cells, w, h, [int(g["seed"])], float(g["density"]))
    sensor.calibrate_collection(cells)
    parts = sensor.reconstruct_from_collection(cells, w, h)
    recs, sens = sensor.export_particles_from_collection(parts)
    m = g["energy"].size
    want = np.empty(m, sensor.PARTICLE_AOS_DTYPE)
    for k in FIELDS + ARRAYS:
        want[k] = g[k]
    assert recs.dtype == sensor.PARTICLE_AOS_DTYPE and recs.tobytes() == want.tobytes()
    cuts = np.concatenate([[0], np.cumsum(g["sensor_lens"].astype(np.int64))])
    assert len(sens) == m
    for i in range(m):
        assert sens[i].tobytes() == g["sensors"][cuts[i]:cuts[i + 1]].tobytes()
    del ev


def _cells_on_device(energy, typ, noisy):
    recs = np.zeros(energy.size, R.SENSOR_AOS_DTYPE)
    recs["energy"], recs["type"] = energy, typ
    recs["calibration_data"]["noisy"] = noisy
    h = aos_collection(sensor.SENSOR_SCHEMA, recs, energy.size)
    d = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    tr.copy_collection(d, h)
    return d


@pytest.mark.parametrize("w,h,events", [(64, 48, 1), (150, 97, 3)])
def test_dense_tied_candidates_vs_oracle(w, h, events):
    """Nearly every cell a candidate, energies drawn from a few values (ties broken by cell index), so
    seeds wait on long blocker chains. The 150 x 97 x 3 case yields more particles than the output's first
    capacity guess, so it also takes the grow-and-write-again path (sk_reco_write)."""
    from paper_2511_04853_b200.devarray import DeviceArray

    rng = np.random.default_rng(w * h)
    n = w * h
    vals = np.array([1.0, 3.0, 6.0, 7.0, 8.0, 50.0, 100.0], np.float32)
    energy = vals[rng.choice(vals.size, n * events, p=[0.05, 0.1, 0.25, 0.2, 0.2, 0.1, 0.1])]
    noise = np.ones(n * events, np.float32)
    typ = rng.integers(0, 4, n * events).astype(np.uint8)
    noisy = rng.random(n * events) < 0.1
    dev = _cells_on_device(energy, typ, noisy)
    parts = sensor.reconstruct_from_collection(dev, w, h, events=events, noise=DeviceArray.from_numpy(noise, CUDA))
    got = _host_particles(parts)
    if events == 3:
        assert len(parts) > max(1024, w * h * events // 200)  # beyond the first guess: written twice
    lo = 0
    starts = np.concatenate([[0], np.cumsum(got["sensor_lens"].astype(np.int64))])
    for i in range(events):
        sl = slice(i * n, (i + 1) * n)
        want = R.reconstruct(energy[sl], noise[sl], typ[sl], noisy[sl], w, h)
        m = parts.event_counts[i]
        assert m == want["energy"].size
        part = {k: got[k][lo:lo + m] for k in FIELDS + ARRAYS + ("sensor_lens",)}
        part["sensors"] = got["sensors"][starts[lo]:starts[lo + m]]
        _compare(part, want, i)
        lo += m


def test_repeated_runs_reuse_the_workspace_and_agree():
    """The device workspace is cached between runs; a bigger batch after a smaller one grows it."""
    small = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(small, 200, 150, [1], 0.004)
    sensor.calibrate_collection(small)
    big = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, CUDA)
    sensor.generate_events(big, 200, 150, [1, 2, 3, 4], 0.004)
    sensor.calibrate_collection(big)
    one = sensor.reconstruct_from_collection(small, 200, 150)
    first = _host_particles(one)
    four = sensor.reconstruct_from_collection(big, 200, 150, events=4)
    again = _host_particles(sensor.reconstruct_from_collection(small, 200, 150))
    _compare(again, first, "again")
    m = four.event_counts[0]
    head = _host_particles(four)
    assert m == len(one)
    for k in FIELDS:
        assert head[k][:m].tobytes() == first[k].tobytes()
