"""Multi-rank host logic on CPU (gloo, world size 2): shard ranges and the one
exchange step of jagged shards."""

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as R
from paper_2511_04853_b200 import shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, lens: np.ndarray, out) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard.shard_range(lens.size, rank, world)
        local = lens[lo:hi].astype(np.int64)
        local_prefix = np.concatenate([[0], np.cumsum(local)])  # each shard scans its own lengths
        offset, total = shard.jagged_shard_offset(int(local_prefix[-1]))
        out[rank] = (lo, hi, shard.rebase_prefix(local_prefix, offset), total)
    finally:
        dist.destroy_process_group()


def test_jagged_shards_rebase_to_the_unsharded_prefix():
    lens = np.random.default_rng(3).integers(0, 21, 1001)
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), lens, out), nprocs=world, join=True)
        res = dict(out)
    full, _ = R.jagged_pack(lens, np.zeros(lens.size, np.int64), np.zeros(int(lens.sum()), np.uint64), np.int64)
    for rank in range(world):
        lo, hi, prefix, total = res[rank]
        assert total == int(lens.sum())
        assert np.array_equal(prefix, full[lo : hi + 1])  # first entry = previous shard's last
    assert res[0][1] == res[1][0]


def test_rebase_wraps_like_the_unsharded_cast():
    # u16 index: the global prefix passes 65535; each shard's rebased prefix must
    # equal the slice of cumsum(int64).astype(u16) (collection.py:553-554)
    lens = np.random.default_rng(5).integers(0, 200, 1500)
    full = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint16)
    cut = 700
    p1 = np.concatenate([[0], np.cumsum(lens[cut:])]).astype(np.uint16)  # shard 1's local prefix, wrapped
    off = int(lens[:cut].sum())
    assert np.array_equal(shard.rebase_prefix(p1, off), full[cut:])
