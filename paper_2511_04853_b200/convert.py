"""Conversion descriptors and the AoSoA / subset / cast extension API.

`plan_desc` turns two layouts of one storage plan into the C-ABI descriptor
(sk_conv_desc) the conversion engine executes: one field per slot of every
main-tag element leaf, located either inside the packed AoS record
(AosLayout.struct_offsets, layouts.py:573-598 byte rules) or at its plane
address (layouts.py:459-460 pitch rule).

The AoSoA tiling with field subset/reorder and per-field cast has no reference
path (SPEC.md:322, 328, 506 list it as a non-goal); it is an extension with
its own API here (`Aosoa`, `to_aosoa`, `from_aosoa`). Its semantics are
defined by oracle/restate.py: tile j holds records [jT, jT+T); inside a tile
each selected field is a contiguous block of T elements in the requested
order and type; casts follow numpy astype (RNE, x86 NaN payload rule); lanes
past the last record are zero.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import layouts as ly
from . import memctx
from .errors import SoakitError, UnsupportedTransferError
from .schema import MAIN_TAG, ROLE_ELEMENT, LeafField, ScalarType

SK_TYPES = nat.TYPE_CODES


def type_code(vt: ScalarType | str) -> int:
    code = vt.storage_code if isinstance(vt, ScalarType) else vt
    return SK_TYPES[code]


def main_slots(layout: ly.LayoutInstance) -> list[tuple[LeafField, int]]:
    """(leaf, slot) for every slot of every main-tag element leaf, plan order."""
    return [(lf, k) for lf in layout.plan.leaves if lf.size_tag == MAIN_TAG and lf.role == ROLE_ELEMENT
            for k in range(lf.extent_multiplier)]


def _is_struct(layout: ly.LayoutInstance, leaf: LeafField) -> bool:
    return isinstance(layout, ly.AosLayout) and leaf.dotted in layout._struct_set


def _side(layout: ly.LayoutInstance):
    """(kind, base pointer, stride) of the main-tag record representation."""
    if isinstance(layout, ly.AosLayout) and layout._struct_buf is not None:
        return nat.KIND_AOS, layout._struct_buf.ptr, layout.record_stride
    return nat.KIND_PLANES, 0, 0


_SLOT_TABLES: dict[int, tuple] = {}


def _slot_table(plan) -> list:
    """(leaf, slot, type code, slot byte offset) of every main-tag record slot, per plan (plans are
    immutable; the descriptor is rebuilt on every transfer, so its static part is computed once)."""
    e = _SLOT_TABLES.get(id(plan))
    if e is None or e[0] is not plan:
        rows = [(lf, k, type_code(lf.value_type), k * lf.value_type.size_bytes)
                for lf in plan.leaves if lf.size_tag == MAIN_TAG and lf.role == ROLE_ELEMENT
                for k in range(lf.extent_multiplier)]
        e = _SLOT_TABLES[id(plan)] = (plan, rows)
    return e[1]


def plan_desc(dst: ly.LayoutInstance, src: ly.LayoutInstance, n: int) -> nat.ConvDesc | None:
    """Descriptor converting records [0, n) of src into dst (same plan)."""
    rows = _slot_table(src.plan)
    if not rows:
        return None
    if len(rows) > nat.MAX_FIELDS:
        raise UnsupportedTransferError(f"plan has {len(rows)} record slots; the engine takes at most {nat.MAX_FIELDS}")
    d = nat.ConvDesc()
    d.n = n
    d.src_kind, d.src, d.src_stride = _side(src)
    d.dst_kind, d.dst, d.dst_stride = _side(dst)
    d.nfields = len(rows)
    s_struct = src._struct_set if isinstance(src, ly.AosLayout) else ()
    d_struct = dst._struct_set if isinstance(dst, ly.AosLayout) else ()
    s_addr = None if s_struct else src.main_slot_addresses([(r[0], r[1]) for r in rows])
    d_addr = None if d_struct else dst.main_slot_addresses([(r[0], r[1]) for r in rows])
    for i, (leaf, k, tc, koff) in enumerate(rows):
        f = d.fields[i]
        f.src_type = f.dst_type = tc
        name = leaf.dotted
        if name in s_struct:
            f.src_off = src.struct_offsets[name] + koff
        else:
            f.src_plane = s_addr[i] if s_addr is not None else src.plane_address(leaf, k)
        if name in d_struct:
            f.dst_off = dst.struct_offsets[name] + koff
        else:
            f.dst_plane = d_addr[i] if d_addr is not None else dst.plane_address(leaf, k)
    return d


def run(desc: nat.ConvDesc, device: int) -> None:
    nat.call("sk_convert", C.byref(desc), device, nat.stream(device))


def plan_info(desc: nat.ConvDesc, device: int = 0) -> dict:
    r, st, mode, grid = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    smem = C.c_size_t()
    nat.call("sk_convert_plan", C.byref(desc), device, C.byref(r), C.byref(st), C.byref(mode), C.byref(smem),
             C.byref(grid))
    return {"records_per_tile": r.value, "stages": st.value, "mode": mode.value & 3, "bulk_in": bool(mode.value & 4),
            "bulk_out": bool(mode.value & 8), "smem_bytes": smem.value, "grid": grid.value}


# ---- AoSoA extension ------------------------------------------------------------------------

@dataclass(frozen=True)
class AosoaField:
    leaf: str           # dotted leaf path (slot 0 of simple arrays: "arr.value")
    dtype: str          # destination storage code ("f32", "i32", ...)
    slot: int = 0


class Aosoa:
    """An array-of-structs-of-arrays image: ceil(n / lanes) tiles of tile_bytes.

    Inside a tile, field i occupies bytes [block_off[i], block_off[i] + lanes *
    itemsize(dtype_i)). The buffer lives in any memory context (cuda by default).
    """

    def __init__(self, n: int, lanes: int, fields: list[AosoaField], info: memctx.ContextInfo | None = None) -> None:
        if lanes < 1 or lanes & (lanes - 1) or lanes > 1024:
            raise SoakitError(f"AoSoA lanes must be a power of two in [1, 1024], got {lanes}")
        self.n = int(n)
        self.lanes = lanes
        self.fields = list(fields)
        self.block_off: list[int] = []
        off = 0
        for f in self.fields:
            self.block_off.append(off)
            off += lanes * np.dtype(_NP[f.dtype]).itemsize
        self.tile_bytes = ly.align_up(off, 16)
        self.ntiles = -(-self.n // lanes)
        self.info = info or memctx.ContextInfo.cuda(0)
        self.buffer = memctx.allocate(self.info, self.ntiles * self.tile_bytes)

    @property
    def nbytes(self) -> int:
        return self.ntiles * self.tile_bytes

    def to_host_bytes(self) -> np.ndarray:
        buf = self.buffer
        if buf._host is not None:
            return np.array(buf._data)
        out = np.empty(buf.length_bytes, dtype=np.uint8)
        if out.size:
            nat.memcpy(out.ctypes.data, buf.ptr, out.size, buf.device)
            nat.sync(buf.device)
        return out

    def free(self) -> None:
        if self.buffer.live:
            memctx.deallocate(self.buffer)


_NP = {"bool": np.bool_, "u8": np.uint8, "u16": np.uint16, "u32": np.uint32, "u64": np.uint64,
       "i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64}


def _aosoa_desc(coll_layout: ly.LayoutInstance, a: Aosoa, to_aosoa: bool) -> nat.ConvDesc:
    d = nat.ConvDesc()
    d.n = a.n
    kind, base, stride = _side(coll_layout)
    a_kind, a_base, a_stride, lanes = nat.KIND_AOSOA, a.buffer.ptr, a.tile_bytes, a.lanes
    if to_aosoa:
        d.src_kind, d.src, d.src_stride = kind, base, stride
        d.dst_kind, d.dst, d.dst_stride, d.dst_lanes = a_kind, a_base, a_stride, lanes
    else:
        d.src_kind, d.src, d.src_stride, d.src_lanes = a_kind, a_base, a_stride, lanes
        d.dst_kind, d.dst, d.dst_stride = kind, base, stride
    d.nfields = len(a.fields)
    for i, af in enumerate(a.fields):
        leaf = coll_layout.plan.leaf(af.leaf)
        if leaf.size_tag != MAIN_TAG or leaf.role != ROLE_ELEMENT:
            raise SoakitError(f"AoSoA fields must be main-tag element leaves, got {af.leaf!r}")
        if not 0 <= af.slot < leaf.extent_multiplier:
            raise SoakitError(f"slot {af.slot} outside leaf {af.leaf!r}")
        f = d.fields[i]
        ctype = type_code(leaf.value_type)
        isz = leaf.value_type.size_bytes
        loc_off = coll_layout.struct_offsets[leaf.dotted] + af.slot * isz if _is_struct(coll_layout, leaf) else 0
        loc_plane = 0 if _is_struct(coll_layout, leaf) else coll_layout.plane_address(leaf, af.slot)
        if to_aosoa:
            f.src_type, f.dst_type = ctype, SK_TYPES[af.dtype]
            f.src_off, f.src_plane = loc_off, loc_plane
            f.dst_off = a.block_off[i]
        else:
            f.src_type, f.dst_type = SK_TYPES[af.dtype], ctype
            f.src_off = a.block_off[i]
            f.dst_off, f.dst_plane = loc_off, loc_plane
    return d


def _engine_device(*infos: memctx.ContextInfo) -> int:
    for info in infos:
        dev = memctx.get_context(info.context).device_of(info.params)
        if dev is not None:
            return dev
    return 0


def to_aosoa(coll, fields: list[AosoaField], lanes: int = 128, out: Aosoa | None = None,
             info: memctx.ContextInfo | None = None, sync: bool = True) -> Aosoa:
    """Convert a collection's records into AoSoA tiles with subset/reorder/cast (K3)."""
    lay = coll.layout
    n = lay.size(MAIN_TAG)
    if out is None:
        out = Aosoa(n, lanes, fields, info)
    elif out.n != n or out.lanes != lanes or out.fields != list(fields):
        raise SoakitError("AoSoA target geometry does not match the request")
    if n:
        dev = _engine_device(out.info, lay.info)
        run(_aosoa_desc(lay, out, True), dev)
        if sync:
            nat.sync(dev)
    return out


def from_aosoa(a: Aosoa, coll, sync: bool = True) -> None:
    """Scatter AoSoA tiles back into a collection (casting to the leaf types)."""
    lay = coll.layout
    with lay.engine_ops():
        # through resize, not the engine's size hook: records of leaves the AoSoA does not carry start at
        # zero and jagged prefix sums stay monotone
        coll.resize(a.n)
    coll._bump()
    if a.n:
        dev = _engine_device(a.info, lay.info)
        run(_aosoa_desc(lay, a, False), dev)
        if sync:
            nat.sync(dev)
