"""GPU jagged-collection packer (K4): prefix sum + member gather.

Reference semantics (collection.py:537-556, transfer.py:297-320):
  prefix[0] = 0, prefix[i+1] = sum(len[:i+1]) computed in int64 and stored
  truncated to the jagged index dtype; pool = concatenation of the segments;
  multi-leaf members split per leaf into separate pools, all leaves sharing
  the segment lengths.

Input here is the image of per-object variable-length vectors: a source pool
of member records (any order, any slack) plus per-record (length, offset)
pairs. `pack` scans the lengths on the device (single-pass decoupled
look-back), resizes the jagged tag to the total, and gathers every member into
the collection's per-leaf pools in record order. Every step runs on the B200;
host-resident collections are staged through device temporaries.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading
from typing import Mapping

import numpy as np

from . import _native as nat
from . import memctx
from .devarray import DeviceArray
from .errors import BoundsError, KindError
from .schema import MAIN_TAG, ROLE_ELEMENT

_NP_CODE = {np.dtype(np.uint8): "u8", np.dtype(np.uint16): "u16", np.dtype(np.uint32): "u32",
            np.dtype(np.uint64): "u64", np.dtype(np.int32): "i32", np.dtype(np.int64): "i64"}


def _as_device(a, dtype, dev: int, keep: list) -> DeviceArray:
    if isinstance(a, DeviceArray):
        if a.device != dev:
            raise KindError(f"device array lives on device {a.device}, packer runs on {dev}")
        return a
    arr = np.ascontiguousarray(a, dtype=dtype) if dtype is not None else np.ascontiguousarray(a)
    d = DeviceArray.from_numpy(arr, memctx.ContextInfo.cuda(dev))
    keep.append(d)
    return d


class _Workspace:
    """Per-device scan scratch (grown on demand), a device total slot and a
    pinned host slot to read it back: no allocations on the per-call path."""

    def __init__(self, dev: int) -> None:
        self.dev = dev
        self.scratch: DeviceArray | None = None
        self.total = DeviceArray(2, np.int64, memctx.ContextInfo.cuda(dev))  # [total, invalid records]
        self.host_total = memctx.allocate(memctx.ContextInfo.pinned(), 16)

    def scratch_for(self, nbytes: int) -> DeviceArray:
        if self.scratch is None or self.scratch.n < nbytes:
            if self.scratch is not None:
                self.scratch.free()
            self.scratch = DeviceArray(max(nbytes, 4096), np.uint8, memctx.ContextInfo.cuda(self.dev))
        return self.scratch


_workspaces: dict[int, _Workspace] = {}

# jagged_fill stages its packed segments here (pinned, so the H2D runs at link speed);
# larger fills use a one-off pageable buffer instead of pinning that much for good
FILL_STAGING_BYTES = int(os.environ.get("SOAKIT_FILL_STAGING_BYTES", str(1 << 30)))


class _FillStaging:
    """One grow-only pinned host area per device for Collection.jagged_fill.
    A fill holds it from packing until its H2D copies have landed (pack() syncs
    before it returns); a concurrent fill on the same device that finds it
    busy packs into pageable memory instead of waiting."""

    def __init__(self) -> None:
        self.lock = threading.Lock()
        self.buf = None

    def alloc(self, nbytes: int):
        if nbytes > FILL_STAGING_BYTES:
            return bytearray(nbytes)
        have = self.buf.length_bytes if self.buf is not None else 0
        if have < nbytes:
            if self.buf is not None:
                memctx.deallocate(self.buf)
                self.buf = None
            self.buf = memctx.allocate(memctx.ContextInfo.pinned(), max(nbytes, 2 * have, 1 << 20))
        return np.frombuffer(self.buf._data, np.uint8, nbytes)


_fill_staging: dict[int, _FillStaging] = {}


@contextlib.contextmanager
def fill_staging(dev: int):
    """Yield an alloc(nbytes) callable for _segpack.pack_segments, or None when
    this device's staging area is in use by another thread."""
    st = _fill_staging.setdefault(dev, _FillStaging())
    if not st.lock.acquire(blocking=False):
        yield None
        return
    try:
        yield st.alloc
    finally:
        st.lock.release()


def _workspace(dev: int) -> _Workspace:
    ws = _workspaces.get(dev)
    if ws is None:
        ws = _workspaces[dev] = _Workspace(dev)
    return ws


def scan(lens: DeviceArray, prefix_ptr: int, prefix_code: str, dev: int, keep: list | None = None) -> int:
    """Exclusive scan of lens into prefix[0..n]; returns the int64 total."""
    n = lens.n
    need = C.c_size_t(0)
    nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
    ws = _workspace(dev)
    scratch = ws.scratch_for(need.value)
    lens_code = _NP_CODE[lens.dtype]
    nat.call("sk_jagged_scan", n, lens.ptr, nat.TYPE_CODES[lens_code], prefix_ptr, nat.TYPE_CODES[prefix_code],
             scratch.ptr, scratch.n, ws.total.ptr, nat.stream(dev))
    nat.memcpy(ws.host_total.ptr, ws.total.ptr, 8, dev)
    nat.sync(dev)
    return int(ws.host_total._data.view(np.int64)[0])


def _check_host_segments(lens, offsets, members: int) -> None:
    """Validate-before-mutate for host inputs (the reference's np.asarray of
    each segment raises before anything changes, collection.py:546)."""
    lens = np.asarray(lens)
    offsets = np.asarray(offsets, dtype=np.int64)
    if lens.size and int(lens.min()) < 0:
        raise BoundsError(f"negative segment length at record {int(np.argmin(lens))}")
    ne = lens > 0
    bad = ne & ((offsets < 0) | (offsets > members - lens.astype(np.int64)))
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        raise BoundsError(f"segment of record {i} ([{offsets[i]}, {offsets[i] + int(lens[i])})) lies outside the "
                          f"source pool of {members} members")


def _validate_on_device(lens_d: DeviceArray, off_d: DeviceArray, members: int, dev: int) -> int:
    """Records whose segment is negative or leaves the pool (sk_jagged_validate), read back."""
    ws = _workspace(dev)
    nat.call("sk_jagged_validate", lens_d.n, lens_d.ptr, nat.TYPE_CODES[_NP_CODE[lens_d.dtype]], off_d.ptr, members,
             ws.total.ptr + 8, nat.stream(dev))
    nat.memcpy(ws.host_total.ptr, ws.total.ptr + 8, 8, dev)
    nat.sync(dev)
    return int(ws.host_total._data.view(np.int64)[0])


def _invalid_segments(bad: int) -> BoundsError:
    return BoundsError(f"{bad} segment(s) have a negative length or lie outside the source pool")


def pack(coll, path: str, lens, src_offsets, src_pool, member_stride: int | None = None,
         member_offsets: Mapping[str, int] | None = None) -> int:
    """Fill jagged vector `path` of `coll` from a member pool; returns the total.

    lens[i] members of record i start at member index src_offsets[i] of
    src_pool (a byte pool of `member_stride`-byte records, or a typed array for
    single-leaf vectors). member_offsets maps each element leaf of the vector
    to its byte offset inside a member record (multi-leaf vectors).
    """
    desc = coll._jagged_desc(path)
    plan = coll.plan
    leaves = [lf for lf in plan.leaves if lf.size_tag == path and lf.role == ROLE_ELEMENT]
    if any(lf.extent_multiplier != 1 for lf in leaves):
        raise KindError(f"multi-slot jagged leaves of {path!r} are not supported")
    n = coll.size()
    lay = coll.layout
    dev = lay.device if lay.device is not None else 0
    keep: list = []
    host_lens = None if isinstance(lens, DeviceArray) else np.asarray(lens)
    keep_type = host_lens is None or (host_lens.dtype in _NP_CODE and host_lens.dtype.kind in "iu")
    lens_d = _as_device(lens, None if keep_type else np.int64, dev, keep)
    if lens_d.n != n:
        raise BoundsError(f"expected {n} segment lengths, got {lens_d.n}")
    off_d = _as_device(src_offsets, np.int64, dev, keep)
    if off_d.n != n:
        raise BoundsError(f"expected {n} segment offsets, got {off_d.n}")
    if member_offsets is None:
        if len(leaves) != 1:
            raise KindError(f"jagged vector {path!r} has {len(leaves)} leaves; pass member_offsets")
        member_offsets = {leaves[0].dotted: 0}
        member_stride = leaves[0].value_type.size_bytes
    if set(member_offsets) != {lf.dotted for lf in leaves}:
        raise KindError(f"member_offsets must name exactly the leaves {[lf.dotted for lf in leaves]}")
    pool_bytes = src_pool.nbytes if isinstance(src_pool, DeviceArray) else np.asarray(src_pool).nbytes
    members = pool_bytes // int(member_stride) if member_stride else 0
    pool_d = _as_device(src_pool, None, dev, keep)
    if not isinstance(lens, DeviceArray) and not isinstance(src_offsets, DeviceArray):
        # host inputs were copied to the device above: validate them there before anything is written
        # (one small kernel instead of a numpy pass over every record; the reference raises before it
        # mutates, collection.py:546)
        bad = _validate_on_device(lens_d, off_d, members, dev)
        if bad:
            for t in keep:
                t.free()
            _check_host_segments(lens, src_offsets, members)  # names the first offending record
            raise _invalid_segments(bad)

    pleaf = plan.leaf(path + ".prefix_sum")
    pcode = pleaf.value_type.storage_code
    psz = pleaf.value_type.size_bytes
    device_resident = not lay.host_visible
    if device_resident:
        prefix_ptr = lay.plane_address(pleaf, 0)
    else:
        tmp_p = DeviceArray(n + 1, pleaf.value_type.np_dtype, memctx.ContextInfo.cuda(dev))
        keep.append(tmp_p)
        prefix_ptr = tmp_p.ptr
    nf = len(leaves)
    offs = (C.c_int64 * nf)(*[member_offsets[lf.dotted] for lf in leaves])
    sizes = (C.c_int32 * nf)(*[lf.value_type.size_bytes for lf in leaves])
    # one launch computes the prefix (into the prefix plane, or a device temp for host-visible layouts),
    # counts invalid device segments and gathers whatever fits the pools' current capacity: a device-resident
    # vector whose pools are large enough is done after one sync; otherwise the prefix is already complete
    # and only the pools have to grow before the gather
    cap = lay.capacity(path) if device_resident else 0
    ws = _workspace(dev)
    need = C.c_size_t(0)
    nat.call("sk_jagged_scratch_bytes", n, C.byref(need))
    starts_bytes = ((cap + 255) // 256 + 1) * 8  # the two-kernel path's work split (one entry per 256 members)
    scratch = ws.scratch_for(-(-need.value // 256) * 256 + starts_bytes)
    ptrs = (C.c_void_p * nf)(*[lay.plane_address(lf, 0) if cap else 0 for lf in leaves])
    nat.call("sk_jagged_pack", n, lens_d.ptr, nat.TYPE_CODES[_NP_CODE[lens_d.dtype]], prefix_ptr,
             nat.TYPE_CODES[pcode], off_d.ptr, pool_d.ptr, members, int(member_stride), nf, offs, sizes, ptrs,
             cap, scratch.ptr, scratch.n, ws.total.ptr, nat.stream(dev))
    nat.memcpy(ws.host_total.ptr, ws.total.ptr, 16, dev)
    nat.sync(dev)
    total, bad = (int(v) for v in ws.host_total._data.view(np.int64)[:2])
    if bad:
        if device_resident:
            # device inputs were checked by the kernel, which already wrote the prefix plane: leave the
            # vector empty and consistent (prefix all zero), then raise
            nat.call("sk_memset_async", prefix_ptr, 0, (n + 1) * psz, nat.stream(dev))
            with lay.engine_ops():
                lay._set_sizes_for_engine({path: 0})
            coll._bump()
            nat.sync(dev)
        for t in keep:
            t.free()
        raise _invalid_segments(bad)
    if device_resident and total <= cap:
        coll._bump()
        with lay.engine_ops():
            lay._set_sizes_for_engine({path: total})
        for t in keep:
            t.free()
        return total
    coll._bump()
    with lay.engine_ops():
        lay.reserve(path, total)
        lay._set_sizes_for_engine({path: total})

    # the scatter needs true positions: if the index dtype wrapped, rescan into int64
    scatter_ptr, scatter_code = prefix_ptr, pcode
    if total >= (1 << (8 * psz - (1 if pcode.startswith("i") else 0))):
        p64 = DeviceArray(n + 1, np.int64, memctx.ContextInfo.cuda(dev))
        keep.append(p64)
        scan(lens_d, p64.ptr, "i64", dev, keep)
        scatter_ptr, scatter_code = p64.ptr, "i64"

    if device_resident:
        dsts = [lay.plane_address(lf, 0) for lf in leaves]
    else:
        tmps = [DeviceArray(total, lf.value_type.np_dtype, memctx.ContextInfo.cuda(dev)) for lf in leaves]
        keep += tmps
        dsts = [t.ptr for t in tmps]
    ptrs = (C.c_void_p * nf)(*dsts)
    nat.call("sk_jagged_scatter", n, scatter_ptr, nat.TYPE_CODES[scatter_code], off_d.ptr, pool_d.ptr,
             int(member_stride), nf, offs, sizes, ptrs, total, nat.stream(dev))
    if not device_resident:
        nat.memcpy(lay.plane_address(pleaf, 0), prefix_ptr, (n + 1) * psz, dev)
        for lf, src in zip(leaves, dsts):
            if total:
                nat.memcpy(lay.plane_address(lf, 0), src, total * lf.value_type.size_bytes, dev)
    nat.sync(dev)
    for t in keep:
        t.free()
    return total
