"""Layout equivalence under random size-changing operation sequences, on the
device (the reference's C2/C3 acceptance gates, test_acceptance.py:154-217,
applied to CUDA-resident per_field / arena / aos collections): after every
operation each device collection dumps identically to a host per_field
collection driven through the same operations."""

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from gpuhelp import CUDA, HOST
from paper_2511_04853_b200 import layouts as ly
from paper_2511_04853_b200 import memctx as mc
from paper_2511_04853_b200 import schema as sc
from paper_2511_04853_b200 import transfer as tr

pytestmark = pytest.mark.gpu

MIXED = sc.Schema("Mixed", (
    sc.declare_per_item("a", sc.F32),
    sc.declare_array("arr", 3, sc.U16),
    sc.declare_jagged("j", sc.I32, sc.F64),
    sc.declare_per_item("b", sc.I64),
    sc.declare_subgroup("g", [sc.declare_per_item("x", sc.BOOL), sc.declare_per_item("y", sc.U8)]),
    sc.declare_global("tot", sc.U32),
))


def _dump_dev(c) -> str:
    h = sk.Collection(c.schema, ly.PER_FIELD, HOST)
    tr.copy_collection(h, c)
    return h.dump()


def _fill_host(c, rng) -> None:
    n = c.size()
    c.column("a").np[:] = rng.standard_normal(n).astype(np.float32)
    c.column("arr").np[:] = rng.integers(0, 65535, (3, n))
    c.column("b").np[:] = rng.integers(-2**40, 2**40, n)
    c.column("g.x").np[:] = rng.integers(0, 2, n).astype(bool)
    c.column("g.y").np[:] = rng.integers(0, 255, n)
    c.jagged_fill("j", [rng.standard_normal(rng.integers(0, 4)) for _ in range(n)])
    c.set_global("tot", int(rng.integers(0, 2**32)))


@pytest.mark.parametrize("seed", range(6))
def test_random_operation_sequences_match_host(seed):
    rng = np.random.default_rng(seed)
    host = sk.Collection(MIXED, ly.PER_FIELD, HOST)
    devs = [sk.Collection(MIXED, ly.PER_FIELD, CUDA), sk.Collection(MIXED, ly.AOS, CUDA),
            sk.Collection(MIXED, ly.ARENA, CUDA, ly.ArenaSpec({sc.MAIN_TAG: 128, "j": 1024}))]
    host.resize(int(rng.integers(1, 20)))
    _fill_host(host, rng)
    for d in devs:
        tr.copy_collection(d, host)
    for step in range(40):
        op = rng.choice(["resize", "insert", "erase", "jresize", "clear", "reload"])
        n = host.size()
        if op == "resize":
            args = (int(rng.integers(0, 40)),)
        elif op == "insert":
            args = (int(rng.integers(0, n + 1)), int(rng.integers(0, 5)))
        elif op == "erase":
            if n == 0:
                continue
            i = int(rng.integers(0, n))
            args = (i, int(rng.integers(0, n - i + 1)))
        elif op == "jresize":
            if n == 0:
                continue
            args = (int(rng.integers(0, n)), int(rng.integers(0, 6)))
        if op == "reload":
            _fill_host(host, rng)
            for d in devs:
                tr.copy_collection(d, host)
        else:
            targets = [(host, mc.HOST)] + [(d, mc.CUDA) for d in devs]
            for c, scope in targets:
                with mc.execution_scope(scope):
                    if op == "resize":
                        c.resize(*args)
                    elif op == "insert":
                        c.insert_records(*args)
                    elif op == "erase":
                        c.erase_records(*args)
                    elif op == "jresize":
                        c.jagged_resize("j", *args)
                    else:
                        c.clear()
        want = host.dump()
        for d in devs:
            assert _dump_dev(d) == want, (seed, step, op, d.kind)
        # prefix invariant (test_acceptance.py:178-189): exclusive running total from zero
        with mc.execution_scope(mc.CUDA):
            p = devs[0].prefix_sums("j")
        assert p[0] == 0 and np.all(np.diff(p.astype(np.int64)) >= 0) and p[-1] == devs[0].jagged_size("j")
