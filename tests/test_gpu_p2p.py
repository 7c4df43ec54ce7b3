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


def _two_gpus() -> bool:
    from paper_2511_04853_b200 import _native as nat

    return nat.device_count() >= 2


@pytest.mark.skipif(not _two_gpus(), reason="needs two GPUs in one process (the gpurun box has one)")
@pytest.mark.parametrize("direction", ["pull", "push"])
def test_in_process_peer_conversion(direction):
    """LOC_PEER inside one process: the AoS records live on cuda:1 and the planes on cuda:0 (pull: the
    kernel on cuda:0 reads cuda:1's HBM over NVLink with TMA bulk copies), or the reverse (push: K2 on
    cuda:0 writes AoS records into cuda:1). Checked byte-exact against the oracle."""
    import paper_2511_04853_b200 as sk
    from oracle import restate as R
    from paper_2511_04853_b200 import layouts as ly, memctx as mc, transfer as tr, workloads as wl

    n = 2_000_003
    recs = wl.obj8_records(n, seed=8)
    host = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.host())
    host.resize(n)
    host.layout._struct_buf._data[: n * 32] = recs.view(np.uint8)
    if direction == "pull":
        far = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.cuda(1))
        tr.copy_collection(far, host)
        near = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(0))
        assert tr.copy_collection(near, far) == "b200-convert"
        back = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, mc.ContextInfo.host())
        tr.copy_collection(back, near)
        want = R.aos_to_planes(recs)
        for i in range(8):
            assert back.column(f"f{i}").np.tobytes() == want[f"f{i}"][0].tobytes()
    else:
        planes = sk.Collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(0))
        tr.copy_collection(planes, host)
        far = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.cuda(1))
        assert tr.copy_collection(far, planes) == "b200-convert"
        back = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.host())
        tr.copy_collection(back, far)
        assert np.array(back.layout._struct_buf._data[: n * 32]).tobytes() == recs.tobytes()
