"""Sharding collections by object index across the GPUs of one box.

Records are independent, so a collection of N records is split into contiguous
ranges [lo, hi) per rank and every rank converts its own range with no data
exchange. The only collective on the path is for jagged collections: each
shard scans its own lengths, then one exclusive scan over the G shard totals
(an all-gather of one int64 per rank) gives each shard the offset to add to
its prefix sums. Layout-changing device-to-device moves between shards pull
the source bytes over NVLink (the conversion kernel reads a peer / IPC-mapped
pointer); same-layout moves are plain peer copies on the copy engines.

torch.distributed is used only as plumbing (rendezvous, one all-gather, the
bench's barrier / max-over-ranks timing).
"""

from __future__ import annotations

import ctypes as C

from . import _native as nat


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous split of [0, n): the first n % world ranks get one extra record."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def exclusive_offsets(totals: list[int]) -> list[int]:
    out, acc = [], 0
    for t in totals:
        out.append(acc)
        acc += int(t)
    return out


def jagged_shard_offset(local_total: int, group=None) -> tuple[int, int]:
    """(offset of this shard's first member, global total) via one all-gather."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = torch.tensor([int(local_total)], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        mine = mine.cuda()
    bufs = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(bufs, mine, group=group)
    totals = [int(b.item()) for b in bufs]
    rank = dist.get_rank(group)
    return exclusive_offsets(totals)[rank], sum(totals)


def rebase_prefix(prefix, offset: int):
    """A shard's local prefix [0, l1, ..] shifted to global positions; its first
    entry equals the previous shard's last. Host arrays: numpy, in the index
    dtype's modular arithmetic (the truncation of local cumsum + offset equals
    the truncation of the global cumsum, collection.py:553-554)."""
    import numpy as np

    prefix = np.asarray(prefix)
    if prefix.dtype.kind in "iu":
        with np.errstate(over="ignore"):
            return (prefix.astype(np.uint64) + np.uint64(offset % (1 << 64))).astype(prefix.dtype)
    return prefix + offset


def global_prefix(coll, path: str, offset: int):
    """The shard's prefix sums of jagged vector `path` rebased by `offset` (from
    jagged_shard_offset): a new array, the collection itself keeps P[0] = 0.
    Device-resident collections get a DeviceArray rebased on the device
    (sk_jagged_rebase); host collections a numpy array."""
    import numpy as np

    from . import memctx
    from .devarray import DeviceArray

    pleaf = coll.plan.leaf(path + ".prefix_sum")
    vt = pleaf.value_type
    n = coll.size()
    lay = coll.layout
    if lay.host_visible:
        return rebase_prefix(np.array(coll.prefix_sums(path), copy=True), offset)
    dev = lay.device
    out = DeviceArray(n + 1, vt.np_dtype, memctx.ContextInfo.cuda(dev))
    nat.memcpy(out.ptr, lay.plane_address(pleaf, 0), (n + 1) * vt.size_bytes, dev)
    nat.call("sk_jagged_rebase", n + 1, out.ptr, nat.TYPE_CODES[vt.storage_code], int(offset), nat.stream(dev))
    nat.sync(dev)
    return out


def pack_sharded(coll, path: str, lens, src_offsets, src_pool, group=None, **member_layout):
    """SURVEY 8e for jagged collections: pack this rank's shard locally (K4),
    one all-gather of the shard totals, then the shard's global prefix.
    Returns (global prefix of this shard, member offset, global total)."""
    from . import jagged

    local = jagged.pack(coll, path, lens, src_offsets, src_pool, **member_layout)
    offset, total = jagged_shard_offset(local, group)
    return global_prefix(coll, path, offset), offset, total


# ---- whole collections across processes (layout-changing peer pulls) ----------------------

def export_collection(coll) -> dict:
    """Picklable description of a device collection allocated with
    ContextInfo.cuda(dev, ipc=True): kind, sizes, capacities and one IPC
    handle per buffer. The owner must keep the collection alive (and its sizes
    unchanged) while importers use it."""
    from . import memctx

    if coll.info.context != memctx.CUDA or not coll.info.params.get("ipc", False):
        raise ValueError("export needs a collection on ContextInfo.cuda(device, ipc=True)")
    lay = coll.layout
    bufs = [(ipc_handle(b.ptr) if b.ptr else b"", b.length_bytes) for b in lay.buffers()]
    spec = None
    if coll.kind == "arena":
        spec = (dict(lay.arena_spec.capacities), lay.arena_spec.alignment)
    return {"kind": coll.kind, "sizes": dict(lay._sizes), "caps": dict(lay._caps), "buffers": bufs,
            "arena": spec, "owner_device": lay.device}


def import_collection(schema, exported: dict, device: int):
    """A collection on this process's `device` whose buffers are the exported
    ones, mapped through CUDA IPC (context cuda_ipc). Layout-changing copies
    out of it run on `device` and pull the bytes over NVLink (or locally when
    both processes share the GPU). free() unmaps."""
    from . import layouts as ly
    from . import memctx
    from .collection import Collection

    arena = ly.ArenaSpec(exported["arena"][0], exported["arena"][1]) if exported["arena"] else None
    coll = Collection(schema, exported["kind"], memctx.ContextInfo.cuda(device), arena)
    lay = coll.layout
    for b in lay.buffers():  # the zero-capacity placeholders
        memctx.deallocate(b)
    info = memctx.ContextInfo(memctx.CUDA_IPC, {"device_id": device})
    ctx = memctx.get_context(memctx.CUDA_IPC)
    adopted = [ctx.adopt(info, ipc_open(device, h) if h else 0, n) for h, n in exported["buffers"]]
    lay._rebind_buffers(adopted)
    lay.info = info
    lay.capabilities = lay._build_capabilities()
    lay._caps = dict(exported["caps"])
    lay._sizes = dict(exported["sizes"])
    coll._bump()
    return coll


# ---- IPC handles for cross-process peer pulls -----------------------------------------

def ipc_handle(dev_ptr: int) -> bytes:
    size = C.c_size_t(0)
    nat.call("sk_ipc_handle_size", C.byref(size))
    buf = (C.c_uint8 * size.value)()
    nat.call("sk_ipc_get_handle", dev_ptr, buf)
    return bytes(buf)


def ipc_open(device: int, handle: bytes) -> int:
    out = C.c_void_p(0)
    raw = (C.c_uint8 * len(handle)).from_buffer_copy(handle)
    nat.call("sk_ipc_open_handle", device, raw, C.byref(out))
    return out.value or 0


def ipc_close(device: int, ptr: int) -> None:
    nat.call("sk_ipc_close_handle", device, ptr)
