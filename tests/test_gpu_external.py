"""External record import/export (transfer.py:246-346) with device-resident
collections; multi-leaf jagged members against the reference's golden
import_external pools."""

from dataclasses import dataclass, field

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, HOST
from paper_2511_04853_b200 import layouts as ly, memctx as mc, sensor, workloads as wl
from skhelp import golden

pytestmark = pytest.mark.gpu


@dataclass
class Hit:
    seed: int
    adc: list = field(default_factory=list)
    t: list = field(default_factory=list)


HIT_BINDING = sk.ExternalBinding(
    extractors={"seed": lambda r: r.seed, "hits.adc": lambda r: r.adc, "hits.t": lambda r: r.t},
    factory=lambda row: Hit(row["seed"], row["hits.adc"], row["hits.t"]))


@pytest.mark.parametrize("kind", [ly.PER_FIELD, ly.AOS])
def test_multi_leaf_import_matches_reference_and_round_trips(kind):
    g = golden("jagged.npz")
    lens = g["hits:lens"].astype(np.int64)
    cuts = np.concatenate([[0], np.cumsum(lens)])
    recs = [Hit(i, g["hits:adc_in"][cuts[i]:cuts[i + 1]].tolist(), g["hits:t_in"][cuts[i]:cuts[i + 1]].tolist())
            for i in range(lens.size)]
    c = sk.Collection(wl.CLUSTER2_SCHEMA, kind, CUDA)
    sk.import_external(c, HIT_BINDING, recs)
    with mc.execution_scope(mc.CUDA):
        assert c.prefix_sums("hits").tobytes() == g["hits:prefix"].tobytes()
        assert c.column("hits.adc").read().tobytes() == g["hits:adc"].tobytes()
        assert c.column("hits.t").read().tobytes() == g["hits:t"].tobytes()
    back = sk.export_external(c, HIT_BINDING)
    assert [(b.seed, b.adc) for b in back] == [(r.seed, r.adc) for r in recs]
    assert all(np.array_equal(np.float32(b.t), np.float32(r.t)) for b, r in zip(back, recs))


def test_particle_import_export_identity():
    rng = np.random.default_rng(4)
    names = ("energy", "x", "y", "origin", "sensors.value", "x_variance", "y_variance", "significance.value",
             "E_contribution.value", "noisy_count.value")
    recs = []
    for i in range(257):
        recs.append({"energy": float(np.float32(rng.standard_normal())), "x": 1.5, "y": -2.0, "origin": i * 7,
                     "sensors.value": rng.integers(0, 2**63, rng.integers(0, 5)).tolist(), "x_variance": 0.25,
                     "y_variance": 0.5, "significance.value": [1.0, 2.0, 3.0, 4.0],
                     "E_contribution.value": [0.5] * 4, "noisy_count.value": [1, 2, 3, 4]})
    binding = sk.ExternalBinding(extractors={k: (lambda r, k=k: r[k]) for k in names}, factory=dict)
    c = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, CUDA)
    sk.import_external(c, binding, recs)
    assert sk.export_external(c, binding) == recs


def test_unbound_leaf_is_reported_first_in_plan_order():
    binding = sk.ExternalBinding(extractors={"seed": lambda r: 0})
    with pytest.raises(sk.UnboundLeafError):
        sk.import_external(sk.Collection(wl.CLUSTER2_SCHEMA, ly.PER_FIELD, HOST), binding, [])
