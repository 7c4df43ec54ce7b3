"""The B200 engine plugged into the reference package itself (soakit 0.1.0).

`install()` registers, through soakit's own public registries and nothing
else, everything a soakit user needs to run the hot path on a B200:

  memory contexts  "cuda" (HBM, param device_id) and "pinned" (page-locked
                   host), via memctx.register_memory_context (memctx.py:269)
  copiers          every ordered pair among host / mockdev / pinned / cuda
                   that involves a new context, via memctx.register_copier
                   (memctx.py:338): cudaMemcpyAsync, or an overlap-safe move
                   for same-buffer ranges (the memmove contract, 314-316)
  transfer spec    "b200-convert" at TransferPriority.EXACT_PAIR via
                   transfer.register_transfer (transfer.py:67-77): AoS <->
                   per_field/arena when an endpoint is cuda or pinned; one
                   launch of the conversion engine for the main-tag leaves,
                   plane copies for prefix sums / jagged pools / globals
  behaviors        "sensor_funcs" re-registered (behaviors.py:46-62,
                   replace=True) with both targets: cuda-resident collections
                   and records run K5 on the device, everything else keeps
                   the reference's numpy functions (detector/schemas.py:15-41)

soakit's own copy_collection, move_collection, Collection size operations,
update_memory_context_info and coll.funcs.* then reach the B200 unmodified.
Device buffers carry a `_DeviceBytes` in `Buffer._data`: it has the byte
length soakit's bookkeeping reads and raises soakit's AccessError on any
attempt to index device memory from Python.

Divergences, by design: get_noise() on a cuda collection returns a host
numpy array (the reference's type) computed on the device, in page-locked
memory that is recycled once the caller drops it; host <-> host and
mockdev pairs stay on the reference's CPU path (the plugin takes only pairs
with a cuda or pinned endpoint). INTEGRATION.md shows the same registration
as a maintainer would write it.
"""

from __future__ import annotations

import ctypes as C
import importlib

import numpy as np

from . import _native as nat
from . import errors as E

CUDA = "cuda"
PINNED = "pinned"

_TYPE = {np.dtype(np.bool_): "bool", np.dtype(np.uint8): "u8", np.dtype(np.uint16): "u16",
         np.dtype(np.uint32): "u32", np.dtype(np.uint64): "u64", np.dtype(np.int32): "i32",
         np.dtype(np.int64): "i64", np.dtype(np.float32): "f32", np.dtype(np.float64): "f64"}

_installed: dict = {}


class _DeviceBytes:
    """Stand-in for Buffer._data of device memory: size and address only."""

    __slots__ = ("ptr", "nbytes", "device")

    def __init__(self, ptr: int, nbytes: int, device: int) -> None:
        self.ptr, self.nbytes, self.device = ptr, nbytes, device

    def __getitem__(self, key):
        raise _soakit().errors.AccessError("device memory has no host view; copy the collection to a host context")

    __setitem__ = __getitem__

    def __len__(self) -> int:
        return self.nbytes


def _soakit():
    return importlib.import_module("soakit")


def _translate(exc: E.SoakitError):
    """The same failure as soakit's exception type (errors share their names)."""
    errors = _soakit().errors
    return getattr(errors, type(exc).__name__, errors.MemoryContextError)(str(exc))


def _native(fn, *args):
    try:
        return fn(*args)
    except E.SoakitError as exc:
        raise _translate(exc) from exc


def _address(buf) -> int:
    data = buf._data
    return data.ptr if isinstance(data, _DeviceBytes) else data.ctypes.data


def _device_of(buf) -> int | None:
    return buf._data.device if isinstance(buf._data, _DeviceBytes) else None


def _make_contexts(smc):
    class CudaContext(smc.MemoryContext):
        """B200 HBM as a soakit memory context (replaces mockdev, memctx.py:164-202)."""

        name = CUDA
        accessible_from = frozenset({CUDA})

        def validate_params(self, params):
            extra = set(params) - {"device_id"}
            if extra:
                raise smc.MemoryContextError(f"cuda does not understand parameters {sorted(extra)}")
            dev = params.get("device_id", 0)
            if isinstance(dev, bool) or not isinstance(dev, int) or dev < 0:
                raise smc.MemoryContextError(f"cuda device_id must be a non-negative integer, got {dev!r}")

        def retag_benign(self, old, new):
            return old.get("device_id", 0) == new.get("device_id", 0)

        def allocate(self, info, nbytes):
            if nbytes < 0:
                raise smc.AllocationError(f"negative allocation size {nbytes}")
            self.validate_params(info.params)
            self.check_capacity(nbytes)
            dev = info.params.get("device_id", 0)
            ptr = _native(nat.malloc, dev, nbytes) if nbytes else 0
            buf = super().allocate(info, 0)  # handle, live registry and counters, as soakit does them
            buf._data = _DeviceBytes(ptr, int(nbytes), dev)
            buf.length_bytes = int(nbytes)
            return buf

        def deallocate(self, buffer):
            data = buffer._data
            super().deallocate(buffer)
            if isinstance(data, _DeviceBytes) and data.ptr:
                _native(nat.free, data.device, data.ptr)

        def memset(self, buffer, byte, offset=0, count=None):
            smc._require_live(buffer, self.name)
            count = buffer.length_bytes - offset if count is None else count
            if not 0 <= byte <= 255:
                raise smc.MemoryContextError(f"memset byte {byte} outside [0, 255]")
            smc._check_range(buffer, offset, count, "memset")
            if count:
                dev = buffer._data.device
                _native(nat.memset, buffer._data.ptr + offset, byte, count, dev)
                _native(nat.sync, dev)
            smc._stats.memsets += 1

    class PinnedContext(smc.MemoryContext):
        """Page-locked host memory: host-visible numpy bytes that DMA at link speed."""

        name = PINNED
        accessible_from = frozenset({smc.HOST})

        def allocate(self, info, nbytes):
            if nbytes < 0:
                raise smc.AllocationError(f"negative allocation size {nbytes}")
            self.validate_params(info.params)
            buf = super().allocate(info, 0)
            if nbytes:
                ptr = _native(nat.host_alloc_pinned, nbytes)
                buf._data = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(ptr))
                buf.length_bytes = int(nbytes)
            return buf

        def deallocate(self, buffer):
            data = buffer._data
            super().deallocate(buffer)
            if data.nbytes:
                _native(nat.host_free_pinned, data.ctypes.data)

    return CudaContext(), PinnedContext()


def _copier(dst, dst_offset, src, src_offset, count) -> None:
    """Native byte copy for any pair with a cuda or pinned endpoint; same
    buffer -> overlap-safe move (memctx.py:356-357). Completes before return."""
    if not count:
        return
    s_dev, d_dev = _device_of(src), _device_of(dst)
    dev = d_dev if d_dev is not None else (s_dev if s_dev is not None else 0)
    if s_dev is not None and d_dev is not None and s_dev != d_dev:
        _native(nat.sync, s_dev)
    move = nat.memmove if src is dst else nat.memcpy
    _native(move, _address(dst) + dst_offset, _address(src) + src_offset, count, dev)
    _native(nat.sync, dev)


def _engine_device(*colls) -> int:
    for c in colls:
        if c.info.context == CUDA:
            return c.info.params.get("device_id", 0)
    return 0


def _conversion_desc(dl, sl, n: int):
    """sk_conv_desc for records [0, n): one field per slot of every main-tag
    element leaf, inside the packed record (AosLayout._struct_dtype offsets,
    layouts.py:573-598) or at its plane (_plane_region, layouts.py:459-460)."""
    S = _soakit()
    slots = [(lf, k) for lf in sl.plan.leaves if lf.size_tag == S.schema.MAIN_TAG and lf.role == S.schema.ROLE_ELEMENT
             for k in range(lf.extent_multiplier)]
    if len(slots) > nat.MAX_FIELDS:
        raise S.errors.UnsupportedTransferError(f"{len(slots)} record slots; the engine takes {nat.MAX_FIELDS}")
    d = nat.ConvDesc()
    d.n = n
    d.nfields = len(slots)

    def side(lay):
        if isinstance(lay, S.layouts.AosLayout):
            return nat.KIND_AOS, _address(lay._struct_buf), lay.record_stride
        return nat.KIND_PLANES, 0, 0

    d.src_kind, d.src, d.src_stride = side(sl)
    d.dst_kind, d.dst, d.dst_stride = side(dl)
    for f, (leaf, k) in zip(d.fields, slots):
        code = nat.TYPE_CODES[_TYPE[np.dtype(leaf.value_type.np_dtype)]]
        f.src_type = f.dst_type = code
        isz = leaf.value_type.size_bytes
        for lay, is_src in ((sl, True), (dl, False)):
            if isinstance(lay, S.layouts.AosLayout):
                off = lay._struct_dtype.fields[leaf.dotted][1] + k * isz
                setattr(f, "src_off" if is_src else "dst_off", off)
            else:
                buf, base = lay._plane_region(leaf, k)
                setattr(f, "src_plane" if is_src else "dst_plane", _address(buf) + base)
    return d


def _is_aos(c) -> bool:
    return c.kind == "aos" and c.layout._struct_buf is not None


def _convert_applies(dst, src) -> bool:
    smc = _soakit().memctx
    ends = {src.info.context, dst.info.context}
    if not ends & {CUDA, PINNED} or not ends <= {smc.HOST, PINNED, CUDA}:
        return False
    return _is_aos(src) != _is_aos(dst)


def _convert_execute(dst, src, opts=None) -> None:
    """transfer.py:171-236 on the B200: reserve + sizes first (capacity errors
    before any write, 177-180), one conversion launch, side leaves as plane
    copies (221-224)."""
    S = _soakit()
    sl, dl = src.layout, dst.layout
    with dl.engine_ops():
        for tag in sl.tags():
            dl.reserve(tag, sl.size(tag))
        dl._set_sizes_for_engine({tag: sl.size(tag) for tag in sl.tags()})
    n = sl.size(S.schema.MAIN_TAG)
    dev = _engine_device(dst, src)
    if n:
        desc = _conversion_desc(dl, sl, n)
        _native(nat.call, "sk_convert", C.byref(desc), dev, nat.stream(dev))
        _native(nat.sync, dev)
    for leaf in sl.plan.leaves:
        if leaf.size_tag == S.schema.MAIN_TAG and leaf.role == S.schema.ROLE_ELEMENT:
            continue
        rows = sl.plane_len(leaf)
        for k in range(sl.plane_count(leaf) if rows else 0):
            s_buf, s_off = sl._plane_region(leaf, k)
            d_buf, d_off = dl._plane_region(leaf, k)
            S.memctx.memcopy_with_context(d_buf, d_off, s_buf, s_off, rows * leaf.value_type.size_bytes, opts)


# ---- the case-study behaviors on cuda-resident sensor collections ------------------------------

_COLS = ("counts", "energy", "calibration_data.noisy", "calibration_data.parameter_A",
         "calibration_data.parameter_B", "calibration_data.noise_A", "calibration_data.noise_B")


def _planes(coll) -> tuple[int, list[int]]:
    lay = coll.layout
    if coll.kind == "aos":
        raise _soakit().errors.UnsupportedTransferError(
            "the B200 case-study kernel reads per_field/arena planes; copy the AoS collection into one first")
    addr = [_address(b) + off for b, off in (lay._plane_region(coll.plan.leaf(c), 0) for c in _COLS)]
    return coll.info.params.get("device_id", 0), addr


def _calibrate_on_device(coll, first: int, count: int) -> None:
    dev, (counts, energy, _, a, b, _, _) = _planes(coll)
    if count:
        _native(nat.call, "sk_sensor_calibrate", count, counts + 8 * first, a + 4 * first, b + 4 * first,
                energy + 4 * first, nat.stream(dev))
        _native(nat.sync, dev)


def _noise_on_device(coll, first: int, count: int) -> np.ndarray:
    from .memctx import host_return_array

    dev, (_, energy, noisy, _, _, na, nb) = _planes(coll)
    out = host_return_array(count, np.float32)  # page-locked, recycled when the caller drops it
    if count:
        tmp = _native(nat.malloc, dev, count * 4)
        try:
            _native(nat.call, "sk_sensor_noise", count, energy + 4 * first, na + 4 * first, nb + 4 * first,
                    noisy + first, tmp, nat.stream(dev))
            _native(nat.memcpy, out.ctypes.data, tmp, count * 4, dev)
            _native(nat.sync, dev)
        finally:
            _native(nat.free, dev, tmp)
    return out


def _sensor_bundle(ref):
    """Dispatchers over the reference's own functions (detector/schemas.py:15-41)."""
    bh = _soakit().behaviors

    def on_device(x) -> bool:
        coll = getattr(x, "_coll", x)
        return coll.info.context == CUDA

    def calibrate_collection(coll):
        return _calibrate_on_device(coll, 0, coll.size()) if on_device(coll) else ref.calibrate_collection(coll)

    def noise_for_collection(coll):
        return _noise_on_device(coll, 0, coll.size()) if on_device(coll) else ref.noise_for_collection(coll)

    def calibrate_object(view):
        return _calibrate_on_device(view._coll, view.index, 1) if on_device(view) else ref._calibrate_object(view)

    def noise_object(view):
        return _noise_on_device(view._coll, view.index, 1)[0] if on_device(view) else ref._noise_object(view)

    return [bh.BehaviorFunction("calibrate_energy", bh.TARGET_OBJECT, calibrate_object),
            bh.BehaviorFunction("calibrate_energy", bh.TARGET_COLLECTION, calibrate_collection),
            bh.BehaviorFunction("get_noise", bh.TARGET_OBJECT, noise_object),
            bh.BehaviorFunction("get_noise", bh.TARGET_COLLECTION, noise_for_collection)]


def install() -> dict:
    """Register the B200 contexts, copiers, transfer spec and behaviors into
    soakit (idempotent). Returns what was registered."""
    if _installed:
        return _installed
    S = _soakit()
    smc, st = S.memctx, S.transfer
    cuda, pinned = _make_contexts(smc)
    smc.register_memory_context(cuda)
    smc.register_memory_context(pinned)
    names = [smc.HOST, smc.MOCKDEV, PINNED, CUDA]
    pairs = []
    for s in names:
        for d in names:
            if {s, d} & {CUDA, PINNED}:
                smc.register_copier(s, d, _copier)
                pairs.append((s, d))
    st.register_transfer("b200-convert", st.TransferPriority.EXACT_PAIR, _convert_applies, _convert_execute)
    ref = importlib.import_module("soakit.detector.schemas")  # registers the reference bundle first
    S.behaviors.register_bundle("sensor_funcs", _sensor_bundle(ref), replace=True)
    _installed.update(contexts=[CUDA, PINNED], copiers=pairs, transfers=["b200-convert"], bundles=["sensor_funcs"])
    return _installed


def cuda_info(device_id: int = 0):
    """soakit ContextInfo of B200 HBM (the plugin's analogue of ContextInfo.mockdev())."""
    return _soakit().memctx.ContextInfo(CUDA, {"device_id": device_id})


def pinned_info():
    return _soakit().memctx.ContextInfo(PINNED)
