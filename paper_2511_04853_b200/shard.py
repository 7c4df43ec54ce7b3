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
    entry equals the previous shard's last (numpy/int64 semantics)."""
    return prefix + offset


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
