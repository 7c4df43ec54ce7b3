"""Random schemas through the conversion engine (in the spirit of the
reference's 120-random-schema check, test_schema.py:245-343): for each seeded
random plan (mixed scalar types, fixed arrays, sub-groups, a jagged vector,
odd packed strides), random records go host AoS -> device per_field ->
device AoS -> host, and every plane / the AoS image must be byte-identical
to the oracle. Exercises the word path and the NVRTC-specialised transforms
across many record signatures."""

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, HOST, PINNED, aos_collection, to_host_aos, to_host_planes
from oracle import restate as R
from paper_2511_04853_b200 import convert as cv, layouts as ly, schema as sc, transfer as tr

pytestmark = pytest.mark.gpu

TYPES = [sc.BOOL, sc.U8, sc.U16, sc.U32, sc.U64, sc.I32, sc.I64, sc.F32, sc.F64, sc.enum_type("E", 300)]


def _random_schema(rng, k):
    props = []
    for i in range(int(rng.integers(1, 9))):
        kind = rng.random()
        t = TYPES[int(rng.integers(0, len(TYPES)))]
        if kind < 0.6:
            props.append(sc.declare_per_item(f"p{i}", t))
        elif kind < 0.8:
            props.append(sc.declare_array(f"a{i}", int(rng.integers(1, 5)), t))
        else:
            props.append(sc.declare_subgroup(f"g{i}", [sc.declare_per_item("u", t),
                                                      sc.declare_per_item("v", TYPES[int(rng.integers(0, 9))])]))
    if rng.random() < 0.4:
        props.append(sc.declare_jagged("jv", sc.I32, TYPES[int(rng.integers(1, 9))]))
    return sc.Schema(f"R{k}", tuple(props))


@pytest.mark.parametrize("k", range(24))
def test_random_schema_round_trip(k):
    rng = np.random.default_rng(1000 + k)
    schema = _random_schema(rng, k)
    n = int(rng.integers(1, 3000))
    src = sk.Collection(schema, ly.AOS, PINNED)
    src.resize(n)
    stride = src.layout.record_stride
    raw = rng.integers(0, 256, n * stride, dtype=np.uint8)
    src.layout._struct_buf._data[: n * stride] = raw
    plan = sc.flatten(schema)
    jag = [t for t in plan.jagged_tags()]
    if jag:
        leaf = plan.leaf("jv.value")
        dt = leaf.value_type.np_dtype
        segs = [np.frombuffer(rng.integers(0, 256, int(rng.integers(0, 4)) * dt.itemsize, dtype=np.uint8).tobytes(), dt)
                for _ in range(n)]
        src.jagged_fill("jv", segs)
    # device planes
    dev = sk.Collection(schema, ly.PER_FIELD, CUDA)
    assert tr.copy_collection(dev, src) == "b200-convert"
    planes = to_host_planes(dev)
    recs = raw.view(src.layout._struct_dtype)
    want = R.aos_to_planes(recs)
    for lf, slot in cv.main_slots(src.layout):
        assert planes[f"{lf.dotted}#{slot}"] == want[lf.dotted][slot].tobytes(), (k, lf.dotted, slot)
    # back to AoS on the device, then to the host
    back = sk.Collection(schema, ly.AOS, CUDA)
    tr.copy_collection(back, dev)
    assert to_host_aos(back).tobytes() == raw.tobytes(), k
    h = sk.Collection(schema, ly.PER_FIELD, HOST)
    tr.copy_collection(h, back)
    assert h.dump() == src.dump()
