"""Sharded jagged pack on the device: two gloo ranks sharing one
GPU each pack their shard with K4, exchange one int64, and rebase their prefix
on the device (sk_jagged_rebase). The shards' global prefixes and pools
concatenate to the unsharded reference result, index-dtype wrap included."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, itype, lens, offs, pool, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_04853_b200 as sk
        from paper_2511_04853_b200 import layouts as ly, memctx as mc, schema as sc, shard

        code = {"i32": sc.I32, "u16": sc.U16}[itype]
        schema = sc.Schema("J", (sc.declare_per_item("seed", sc.U64), sc.declare_jagged("members", code, sc.U64)))
        lo, hi = shard.shard_range(lens.size, rank, world)
        c = sk.Collection(schema, ly.PER_FIELD, mc.ContextInfo.cuda(0))
        with mc.execution_scope(mc.CUDA):
            c.resize(hi - lo)
        gp, off, total = shard.pack_sharded(c, "members", lens[lo:hi].astype(np.int64), offs[lo:hi], pool)
        with mc.execution_scope(mc.CUDA):
            members = np.asarray(c.column("members").read()).copy()
        out[rank] = (lo, hi, gp.numpy().copy(), off, total, members)
        gp.free()
        c.free()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("itype,idx", [("i32", np.int32), ("u16", np.uint16)])
def test_sharded_pack_equals_unsharded(itype, idx):
    from oracle import restate as R

    rng = np.random.default_rng(11)
    n = 20_000
    lens = rng.integers(0, 12, n)
    order = rng.permutation(n)
    gaps = lens[order] + rng.integers(0, 3, n)
    offs = np.empty(n, np.int64)
    offs[order] = np.concatenate([[0], np.cumsum(gaps)[:-1]])
    pool = rng.integers(0, 1 << 62, int(gaps.sum()), dtype=np.uint64)
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), itype, lens, offs, pool, out), nprocs=world, join=True)
        res = dict(out)
    prefix, packed = R.jagged_pack(lens, offs, pool, idx)
    assert int(lens.sum()) > 65535  # the u16 case wraps
    got_pool = np.concatenate([res[r][5] for r in range(world)])
    assert got_pool.tobytes() == packed.tobytes()
    for r in range(world):
        lo, hi, gp, off, total, _ = res[r]
        assert total == int(lens.sum())
        assert gp.dtype == prefix.dtype
        assert gp.tobytes() == prefix[lo:hi + 1].tobytes()
