"""Collection-to-collection transfers through a priority-ordered registry.

Same registry contract as soakit/transfer.py (register_transfer 67-77,
resolution by (priority, registration order) 90-91, copy_collection 94-116
returning the chosen spec name, move_collection 119-124). Built-ins:

  b200-convert     EXACT_PAIR. Any pair whose record representations differ
                   (AoS <-> planes) between host/pinned/cuda placements. Main-
                   tag element leaves go through ONE launch of the conversion
                   engine (sk_convert): device-resident endpoints are converted
                   in HBM, host endpoints stream through the chunked H2D |
                   convert | D2H pipeline, a peer-device source is pulled over
                   NVLink. Side leaves (prefix sums, jagged pools, globals) are
                   plane copies. Replaces per-leaf-default (transfer.py:171-236)
                   and lifts its restriction that AoS destinations must be on
                   the host (transfer.py:165-167).
  bulk-same-kind   SAME_LAYOUT_KIND. Identical to the reference
                   (transfer.py:130-146): refit, one copy per buffer.
  plane-copy       PER_LEAF_DEFAULT. Planes on both sides (per_field <->
                   arena, arenas with different specs): one copy per plane on
                   the copy engines.

There is no CPU conversion path: a conversion without a usable B200 raises.
"""

from __future__ import annotations

import ctypes as C
import itertools
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Any, Callable, Mapping

from . import _native as nat
from . import convert as cv
from . import layouts as ly
from . import memctx
from .collection import Collection
from .errors import RegistryError, SchemaMismatchError, TransferError, UnboundLeafError, UnsupportedTransferError
from .schema import MAIN_TAG, ROLE_ELEMENT


class TransferPriority(IntEnum):
    EXACT_PAIR = 0
    SAME_LAYOUT_KIND = 1
    PER_LEAF_DEFAULT = 2


@dataclass(frozen=True)
class TransferSpec:
    name: str
    priority: TransferPriority
    applies: Callable[[Collection, Collection], bool]
    execute: Callable[[Collection, Collection, Mapping[str, Any] | None], None]
    seq: int = field(default=0, compare=False)


_specs: dict[str, TransferSpec] = {}
_seq = itertools.count()
_chosen: dict[str, int] = {}


def chosen_transfer_counts() -> dict[str, int]:
    return dict(_chosen)


def reset_transfer_counts() -> None:
    _chosen.clear()


def register_transfer(name: str, priority: TransferPriority, applies, execute) -> None:
    if name in _specs:
        raise RegistryError(f"transfer spec {name!r} is already registered")
    _specs[name] = TransferSpec(name, TransferPriority(priority), applies, execute, next(_seq))


def unregister_transfer(name: str) -> None:
    if name not in _specs:
        raise RegistryError(f"no transfer spec named {name!r}")
    del _specs[name]


def _ordered() -> list[TransferSpec]:
    return sorted(_specs.values(), key=lambda s: (int(s.priority), s.seq))


def registered_transfers() -> tuple[str, ...]:
    return tuple(s.name for s in _ordered())


def copy_collection(dst: Collection, src: Collection, opts: Mapping[str, Any] | None = None) -> str:
    """Copy src's logical content into dst; returns the name of the spec used."""
    if dst is src or dst.layout is src.layout:
        raise TransferError("source and destination alias the same storage")
    if dst.plan != src.plan:
        raise SchemaMismatchError(f"collections flatten differently: {src.schema.name!r} vs {dst.schema.name!r}")
    for spec in _ordered():
        if spec.applies(dst, src):
            spec.execute(dst, src, opts)
            dst._bump()
            _chosen[spec.name] = _chosen.get(spec.name, 0) + 1
            return spec.name
    raise UnsupportedTransferError(
        f"no transfer applies for ({src.kind}, {src.info.context}) -> ({dst.kind}, {dst.info.context}); "
        f"tried {[s.name for s in _ordered()]}"
    )


def move_collection(dst: Collection, src: Collection, opts: Mapping[str, Any] | None = None) -> str:
    name = copy_collection(dst, src, opts)
    with src.layout.engine_ops():
        src.clear()
    return name


# ---- shared helpers -----------------------------------------------------------------------------

_ENGINE_CONTEXTS = (memctx.HOST, memctx.PINNED, memctx.CUDA, memctx.CUDA_IPC)


def _engine_device(dst: Collection, src: Collection) -> int:
    """The GPU that runs the conversion: the destination's if device-resident,
    else the source's, else device 0 (host <-> host staged through HBM)."""
    for c in (dst, src):
        if c.device is not None:
            return c.device
    return 0


def _match_sizes(dst: Collection, src: Collection) -> None:
    """Reserve then set sizes: capacity errors surface before any write
    (transfer.py:177-180, test_transfer.py:292-300)."""
    sl, dl = src.layout, dst.layout
    with dl.engine_ops():
        for tag in sl.tags():
            dl.reserve(tag, sl.size(tag))
        dl._set_sizes_for_engine({tag: sl.size(tag) for tag in sl.tags()})


def _copy_planes(dst: Collection, src: Collection, leaves, opts) -> None:
    sl, dl = src.layout, dst.layout
    for leaf in leaves:
        n = sl.plane_len(leaf)
        if n == 0:
            continue
        isz = leaf.value_type.size_bytes
        for k in range(sl.plane_count(leaf)):
            s_buf, s_off = sl._plane_region(leaf, k)
            d_buf, d_off = dl._plane_region(leaf, k)
            memctx.memcopy_with_context(d_buf, d_off, s_buf, s_off, n * isz, opts)


def _sync(dst: Collection, src: Collection, opts, engine: int | None = None) -> None:
    if opts and opts.get("async"):
        return
    for dev in {dst.device, src.device, engine} - {None}:
        nat.sync(dev)


# ---- b200-convert ------------------------------------------------------------------------------

def _has_struct(c: Collection) -> bool:
    return isinstance(c.layout, ly.AosLayout) and c.layout._struct_buf is not None


def _convert_applies(dst: Collection, src: Collection) -> bool:
    if src.info.context not in _ENGINE_CONTEXTS or dst.info.context not in _ENGINE_CONTEXTS:
        return False
    return _has_struct(src) != _has_struct(dst)


_desc_cache: dict = {}


def _cached_desc(dl, sl, n):
    """Descriptors are pure functions of the two layouts' buffer addresses,
    capacities and n: reuse them across repeated transfers (host overhead is
    what bounds small conversions)."""
    key = (n, tuple(b.ptr for b in sl.buffers()), tuple(b.ptr for b in dl.buffers()),
           tuple(sl._caps.values()), tuple(dl._caps.values()), type(sl), type(dl), id(sl.plan))
    desc = _desc_cache.get(key)
    if desc is None:
        if len(_desc_cache) > 256:
            _desc_cache.clear()
        desc = _desc_cache[key] = cv.plan_desc(dl, sl, n)
    return desc


def _convert_execute(dst: Collection, src: Collection, opts: Mapping[str, Any] | None = None) -> None:
    fuse = (opts or {}).get("fuse")
    if fuse is not None:
        # copy_collection(dst, src, {"fuse": "sensor_funcs"}): the conversion also runs the bundle's
        # collection behaviors in the same pass (sensor.fused_transfer); unknown bundles are refused
        from . import sensor

        if fuse != "sensor_funcs":
            raise TransferError(f"no fused conversion for behavior bundle {fuse!r}")
        sensor.fused_transfer(dst, src, opts)
        return
    _match_sizes(dst, src)
    sl, dl = src.layout, dst.layout
    memctx.pin_for_transfer(*sl.buffers(), *dl.buffers())
    n = sl.size(MAIN_TAG)
    dev = _engine_device(dst, src)
    desc = _cached_desc(dl, sl, n)
    if desc is not None and n:
        cv.run(desc, dev)
    side = [lf for lf in sl.plan.leaves if not (lf.size_tag == MAIN_TAG and lf.role == ROLE_ELEMENT)]
    _copy_planes(dst, src, side, {"async": True})
    _sync(dst, src, opts, dev)


# ---- bulk-same-kind (transfer.py:130-146) -------------------------------------------------------

def _bulk_applies(dst: Collection, src: Collection) -> bool:
    if src.kind != dst.kind or not memctx.has_copier(src.info.context, dst.info.context):
        return False
    return not (src.kind == ly.ARENA and src.layout.arena_spec != dst.layout.arena_spec)


def _bulk_execute(dst: Collection, src: Collection, opts: Mapping[str, Any] | None = None) -> None:
    sl, dl = src.layout, dst.layout
    with dl.engine_ops():
        dl._refit_for_engine(sl)
    for sb, db in zip(sl.buffers(), dl.buffers()):
        if sb.length_bytes:
            memctx.memcopy_with_context(db, 0, sb, 0, sb.length_bytes, {"async": True})
    _sync(dst, src, opts)


# ---- plane-copy ---------------------------------------------------------------------------------

def _planes_applies(dst: Collection, src: Collection) -> bool:
    return (not _has_struct(src) and not _has_struct(dst)
            and memctx.has_copier(src.info.context, dst.info.context))


def _planes_execute(dst: Collection, src: Collection, opts: Mapping[str, Any] | None = None) -> None:
    _match_sizes(dst, src)
    _copy_planes(dst, src, src.plan.leaves, {"async": True})
    _sync(dst, src, opts)


# ---- prepared transfers: one CUDA-graph launch per repeat ---------------------------------------

class PreparedTransfer:
    """copy_collection(dst, src) captured once into a CUDA graph.

    For transfers repeated between the same two collections (a serving loop,
    per-event staging), the host-side work (spec resolution, descriptor and
    plan, per-chunk copy calls of the host pipeline) is paid once. run()
    replays the whole transfer with one graph launch. The capture runs the
    transfer once eagerly first (allocations, NVRTC, staging), so the graph
    holds only stream work. Valid while neither collection changes size or
    storage; pageable-host endpoints cannot be captured (use pinned)."""

    def __init__(self, dst: Collection, src: Collection) -> None:
        ends = (src.info.context, dst.info.context)
        if memctx.HOST in ends:
            raise TransferError("prepared transfers need pinned or device endpoints: pageable host memory "
                                "cannot be captured into a CUDA graph")
        if all(c == memctx.PINNED for c in ends):
            # pinned <-> pinned byte copies run on the host (numpy), outside any stream: a graph would hold
            # only part of the transfer (or nothing) and replay stale side data
            raise TransferError("prepared transfers need a device endpoint; pinned <-> pinned copies run on the "
                                "host and cannot be replayed from a CUDA graph")
        self.dst, self.src = dst, src
        self.spec = copy_collection(dst, src)  # eager warm-up; also resolves the spec
        self.device = _engine_device(dst, src)
        for dev in {dst.device, src.device, self.device} - {None}:
            nat.sync(dev)
        spec = _specs[self.spec]
        nat.call("sk_capture_begin", self.device)
        graph = C.c_void_p(0)
        try:
            spec.execute(dst, src, {"async": True})
        finally:
            nat.check(nat.lib().sk_capture_end(self.device, C.byref(graph)), "sk_capture_end")
        self.graph = graph.value
        self._geometry = (_geometry(dst), _geometry(src))

    def run(self, sync: bool = True) -> str:
        if self.graph is None:
            raise TransferError("prepared transfer is closed")
        if (_geometry(self.dst), _geometry(self.src)) != self._geometry:
            raise TransferError("prepared transfer is stale: a collection changed size or storage")
        nat.call("sk_graph_launch", self.graph, self.device)
        self.dst._bump()
        if sync:
            nat.sync(self.device)
        return self.spec

    def close(self) -> None:
        if self.graph:
            nat.call("sk_graph_destroy", self.graph)
            self.graph = None

    def __del__(self) -> None:  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass


def _geometry(c: Collection) -> tuple:
    """What a captured graph bakes in: sizes, buffer addresses, capacities."""
    lay = c.layout
    return (tuple(lay._sizes.items()),
            tuple((b.ptr, b.length_bytes) for b in lay.buffers()),
            tuple(lay._caps.values()))


def prepare(dst: Collection, src: Collection) -> PreparedTransfer:
    """Capture copy_collection(dst, src) as a CUDA graph for cheap repeats."""
    return PreparedTransfer(dst, src)


# ---- external record import/export (transfer.py:246-346) ---------------------------------------

@dataclass(frozen=True)
class ExternalBinding:
    """extractors: dotted element-leaf path -> fn(record) -> value (a slot list
    for multi-slot leaves, the whole segment for jagged leaves); factory:
    fn(dict of the same keys) -> new external record, for export."""

    extractors: Mapping[str, Callable[[Any], Any]]
    factory: Callable[[Mapping[str, Any]], Any] | None = None


def _element_leaves(coll: Collection, binding: ExternalBinding):
    element = [lf for lf in coll.plan.leaves if lf.role == ROLE_ELEMENT]
    have = set(binding.extractors)
    for lf in element:  # first hole in plan order
        if lf.dotted not in have:
            raise UnboundLeafError(f"binding has no extractor for leaf {lf.dotted!r}")
    extra = sorted(have - {lf.dotted for lf in element})
    if extra:
        raise TransferError(f"binding names leaves outside the plan: {extra}")
    return element


def import_external(coll: Collection, binding: ExternalBinding, records) -> None:
    """Replace coll's content with external records. Main-tag columns are
    materialised from the Python objects into a host staging collection and
    moved with copy_collection; jagged members go through the GPU packer
    (multi-leaf members as one struct pool split per leaf)."""
    import numpy as np

    from . import jagged as jg
    from .errors import KindError

    element = _element_leaves(coll, binding)
    records = list(records)
    n = len(records)
    stage = Collection(coll.schema, ly.PER_FIELD, memctx.ContextInfo.host())
    stage.resize(n)
    for leaf in element:
        if leaf.size_tag != MAIN_TAG or n == 0:
            continue
        ex = binding.extractors[leaf.dotted]
        col = stage.layout.column_np(leaf)
        dt = leaf.value_type.np_dtype
        if leaf.extent_multiplier == 1:
            col[:] = np.asarray([ex(r) for r in records], dtype=dt)
        else:
            block = np.asarray([list(ex(r)) for r in records], dtype=dt)
            if block.shape != (n, leaf.extent_multiplier):
                raise TransferError(f"extractor for {leaf.dotted!r} produced shape {block.shape}, "
                                    f"expected ({n}, {leaf.extent_multiplier})")
            col[:] = block.T
    segs = {}
    for tag in coll.plan.jagged_tags():
        jleaves = [lf for lf in element if lf.size_tag == tag.id]
        if any(lf.extent_multiplier != 1 for lf in jleaves):
            raise KindError(f"import into multi-slot jagged leaves of {tag.id!r} is not supported")
        per_leaf = {lf.dotted: [np.asarray(list(binding.extractors[lf.dotted](r)), dtype=lf.value_type.np_dtype)
                                for r in records] for lf in jleaves}
        lengths = [a.size for a in per_leaf[jleaves[0].dotted]]
        for lf in jleaves[1:]:
            if [a.size for a in per_leaf[lf.dotted]] != lengths:
                raise TransferError(f"jagged leaves {jleaves[0].dotted!r} and {lf.dotted!r} disagree on "
                                    "segment lengths")
        segs[tag.id] = (jleaves, per_leaf, np.asarray(lengths, np.int64))
    with coll.layout.engine_ops():
        coll.clear()
    copy_collection(coll, stage)
    for path, (jleaves, per_leaf, lengths) in segs.items():
        dt = np.dtype([(lf.dotted, lf.value_type.np_dtype) for lf in jleaves])
        pool = np.empty(int(lengths.sum()), dt)
        for lf in jleaves:
            pool[lf.dotted] = np.concatenate(per_leaf[lf.dotted]) if n else []
        offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]) if n else np.empty(0, np.int64)
        jg.pack(coll, path, lengths, offsets, pool.view(np.uint8), member_stride=dt.itemsize,
                member_offsets={lf.dotted: dt.fields[lf.dotted][1] for lf in jleaves})
    stage.free()


def export_external(coll: Collection, binding: ExternalBinding) -> list:
    """One external record per collection record via binding.factory."""
    element = _element_leaves(coll, binding)
    if binding.factory is None:
        raise TransferError("binding has no factory; cannot export")
    host = coll
    if not coll.layout.host_visible or isinstance(coll.layout, ly.AosLayout):
        host = Collection(coll.schema, ly.PER_FIELD, memctx.ContextInfo.host())
        copy_collection(host, coll)
    cols = {lf.dotted: host.layout.column_np(lf, writable=False) for lf in element}
    prefixes = {t.id: host.prefix_sums(t.id) for t in host.plan.jagged_tags()}
    out = []
    for i in range(host.size()):
        row = {}
        for lf in element:
            col = cols[lf.dotted]
            if lf.size_tag == MAIN_TAG:
                row[lf.dotted] = col[i].item() if lf.extent_multiplier == 1 else col[:, i].tolist()
            else:
                pv = prefixes[lf.size_tag]
                row[lf.dotted] = col[int(pv[i]):int(pv[i + 1])].tolist()
        out.append(binding.factory(row))
    return out


register_transfer("b200-convert", TransferPriority.EXACT_PAIR, _convert_applies, _convert_execute)
register_transfer("bulk-same-kind", TransferPriority.SAME_LAYOUT_KIND, _bulk_applies, _bulk_execute)
register_transfer("plane-copy", TransferPriority.PER_LEAF_DEFAULT, _planes_applies, _planes_execute)
