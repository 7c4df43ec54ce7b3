"""Layout-changing pulls from another process's collection through CUDA IPC
(the multi-GPU path of SURVEY 8e, exercised here with two processes sharing
one GPU: the importer's conversion kernel reads the exporter's buffers)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, port: int, results) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    import paper_2511_04853_b200 as sk
    from paper_2511_04853_b200 import _native as nat, layouts as ly, memctx as mc, sensor, shard, transfer as tr

    try:
        box = [None]
        if rank == 0:
            rng = np.random.default_rng(21)
            n = 3001
            host = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, mc.ContextInfo.host())
            host.resize(n)
            host.layout._struct_buf._data[: n * 64] = rng.integers(0, 256, n * 64, dtype=np.uint8)
            host.jagged_fill("sensors", [rng.integers(0, 2**63, rng.integers(0, 6), dtype=np.uint64)
                                         for _ in range(n)])
            owned = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, mc.ContextInfo.cuda(0, ipc=True))
            tr.copy_collection(owned, host)
            nat.sync(0)
            box = [(shard.export_collection(owned), host.dump())]
        dist.broadcast_object_list(box, src=0)
        if rank == 1:
            exported, want = box[0]
            remote = shard.import_collection(sensor.PARTICLE_SCHEMA, exported, 0)
            local = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(0))
            name = tr.copy_collection(local, remote)  # K1 pulling the exporter's bytes
            back = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, mc.ContextInfo.host())
            tr.copy_collection(back, local)
            results["spec"] = name
            results["equal"] = back.dump() == want
            remote.free()
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_cross_process_layout_changing_pull():
    with mp.Manager() as m:
        results = m.dict()
        mp.spawn(_worker, args=(_port(), results), nprocs=2, join=True)
        res = dict(results)
    assert res["spec"] == "b200-convert"
    assert res["equal"]
