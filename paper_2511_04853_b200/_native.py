"""ctypes binding of libsoakit_b200.so (declared in include/soakit_b200.h).

The library is the product: there is no CPU fallback. If the shared object is
missing, the first native call raises ImportError naming the build step; if no
B200 is present, calls raise MemoryContextError with the CUDA runtime message.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors as E

LIB_PATH = os.environ.get("SK_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                          "libsoakit_b200.so")  # override: A/B builds

# status codes (soakit_b200.h)
SK_OK = 0
SK_ERR_ALLOC = 1
SK_ERR_RANGE = 2
SK_ERR_UNSUPPORTED = 3
SK_ERR_INVALID = 4
SK_ERR_CUDA = 5
SK_ERR_NO_DEVICE = 6

# scalar type codes, schema.py _SCALAR_CODES order
TYPE_CODES = {"bool": 0, "u8": 1, "u16": 2, "u32": 3, "u64": 4, "i32": 5, "i64": 6, "f32": 7, "f64": 8}

KIND_AOS = 0
KIND_PLANES = 1
KIND_AOSOA = 2
MAX_FIELDS = 64


class Field(C.Structure):
    _fields_ = [
        ("src_type", C.c_int32),
        ("dst_type", C.c_int32),
        ("src_off", C.c_int64),
        ("dst_off", C.c_int64),
        ("src_plane", C.c_void_p),
        ("dst_plane", C.c_void_p),
    ]


class ConvDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("src_kind", C.c_int32),
        ("dst_kind", C.c_int32),
        ("src", C.c_void_p),
        ("dst", C.c_void_p),
        ("src_stride", C.c_int64),
        ("dst_stride", C.c_int64),
        ("src_lanes", C.c_int32),
        ("dst_lanes", C.c_int32),
        ("nfields", C.c_int32),
        ("flags", C.c_int32),
        ("fields", Field * MAX_FIELDS),
    ]


class RecoOut(C.Structure):
    """sk_reco_out: the per_field planes a reconstruction writes into."""
    _fields_ = [
        ("energy", C.c_void_p),
        ("x", C.c_void_p),
        ("y", C.c_void_p),
        ("origin", C.c_void_p),
        ("x_variance", C.c_void_p),
        ("y_variance", C.c_void_p),
        ("significance", C.c_void_p * 4),
        ("e_contribution", C.c_void_p * 4),
        ("noisy_count", C.c_void_p * 4),
        ("sensor_prefix", C.c_void_p),
        ("sensor_prefix_type", C.c_int),
        ("sensor_pool", C.c_void_p),
        ("particle_capacity", C.c_int64),
        ("pool_capacity", C.c_int64),
    ]


_P = C.c_void_p
_U = C.c_size_t
_I = C.c_int
_I64 = C.c_int64
_SZ = C.c_size_t

# name -> argtypes (restype is int for all but sk_last_error)
_SIGNATURES = {
    "sk_version": [],
    "sk_device_count": [C.POINTER(_I)],
    "sk_device_info": [_I, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), C.POINTER(_SZ)],
    "sk_malloc": [_I, _SZ, C.POINTER(_P)],
    "sk_free": [_I, _P],
    "sk_host_alloc_pinned": [_SZ, C.POINTER(_P)],
    "sk_host_free_pinned": [_P],
    "sk_host_register": [_P, _SZ],
    "sk_host_unregister": [_P],
    "sk_stream_default": [_I, C.POINTER(_U)],
    "sk_stream_sync": [_U],
    "sk_device_sync": [_I],
    "sk_event_create": [C.POINTER(_U)],
    "sk_event_destroy": [_U],
    "sk_event_record": [_U, _U],
    "sk_event_elapsed_ms": [_U, _U, C.POINTER(C.c_float)],
    "sk_memset_async": [_P, _I, _SZ, _U],
    "sk_memcpy_async": [_P, _P, _SZ, _U],
    "sk_memmove_async": [_P, _P, _SZ, _U],
    "sk_peer_enable": [_I, _I],
    "sk_convert": [C.POINTER(ConvDesc), _I, _U],
    "sk_convert_plan": [C.POINTER(ConvDesc), _I, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), C.POINTER(_SZ),
                        C.POINTER(_I)],
    "sk_convert_specialize_check": [C.POINTER(ConvDesc), C.POINTER(_I), C.c_char_p, _SZ, C.POINTER(_SZ)],
    "sk_capture_begin": [_I],
    "sk_capture_end": [_I, C.POINTER(_P)],
    "sk_graph_launch": [_P, _I],
    "sk_graph_destroy": [_P],
    "sk_jagged_scratch_bytes": [_I64, C.POINTER(_SZ)],
    "sk_jagged_scan": [_I64, _P, _I, _P, _I, _P, _SZ, _P, _U],
    "sk_jagged_scatter": [_I64, _P, _I, _P, _P, _I64, _I, C.POINTER(_I64), C.POINTER(C.c_int32), C.POINTER(_P),
                          _I64, _U],
    "sk_jagged_pack": [_I64, _P, _I, _P, _I, _P, _P, _I64, _I64, _I, C.POINTER(_I64), C.POINTER(C.c_int32),
                       C.POINTER(_P), _I64, _P, _SZ, _P, _U],
    "sk_jagged_validate": [_I64, _P, _I, _P, _I64, _P, _U],
    "sk_jagged_rebase": [_I64, _P, _I, _I64, _U],
    "sk_jagged_trace": [_P, _SZ],
    "sk_sensor_calibrate": [_I64, _P, _P, _P, _P, _U],
    "sk_sensor_noise": [_I64, _P, _P, _P, _P, _P, _U],
    "sk_sensor_convert_calibrate": [C.POINTER(ConvDesc), _I, _I, _I, _I, _I, _I, _I, _P, _I, _U],
    "sk_sensor_generate": [_I64, _I64, C.POINTER(C.c_uint64), _I, _I64, C.POINTER(C.c_double), _P, _P, _P, _P, _P,
                           _P, _P, _P, _U],
    "sk_reco_run": [_I64, _I64, _I, _P, _P, _P, _P, C.POINTER(RecoOut), _I, _U, C.POINTER(_P), C.POINTER(_I64),
                    C.POINTER(_I64), C.POINTER(_I), C.POINTER(_I)],
    "sk_reco_event_counts": [_P, C.POINTER(_I64)],
    "sk_reco_write": [_P, C.POINTER(RecoOut), _U],
    "sk_reco_free": [_P, _U],
    "sk_fill_random": [_P, _SZ, C.c_uint64, C.c_uint64, _U],
    "sk_compare_bytes": [_P, _P, _SZ, _P, _U],
    "sk_move_batch_async": [_P, _I, _U],
    "sk_malloc_shareable": [_I, _SZ, C.POINTER(_P)],
    "sk_free_shareable": [_I, _P],
    "sk_ipc_handle_size": [C.POINTER(_SZ)],
    "sk_ipc_get_handle": [_P, _P],
    "sk_ipc_open_handle": [_I, _P, C.POINTER(_P)],
    "sk_ipc_close_handle": [_I, _P],
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libsoakit_b200.so once; raise ImportError if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA extension is required (no CPU fallback). "
                "Run `python -c 'import __graft_entry__ as g; g.build()'` or `make -C paper_2511_04853_b200/csrc`."
            )
        handle = C.CDLL(LIB_PATH)
        handle.sk_last_error.restype = C.c_char_p
        handle.sk_last_error.argtypes = []
        for name, args in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = C.c_int
            fn.argtypes = args
        _lib = handle
        return _lib


def exported_names() -> list[str]:
    return ["sk_last_error", *_SIGNATURES]


_EXC = {
    SK_ERR_ALLOC: E.AllocationError,
    SK_ERR_RANGE: E.CopyError,
    SK_ERR_UNSUPPORTED: E.UnsupportedTransferError,
    SK_ERR_INVALID: E.SoakitError,
    SK_ERR_CUDA: E.MemoryContextError,
    SK_ERR_NO_DEVICE: E.MemoryContextError,
}


def check(status: int, what: str = "") -> None:
    if status == SK_OK:
        return
    msg = lib().sk_last_error().decode(errors="replace")
    exc = _EXC.get(status, E.SoakitError)
    raise exc(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


# ---- small conveniences ---------------------------------------------------------

_streams: dict[int, int] = {}


def device_count() -> int:
    n = C.c_int(0)
    st = lib().sk_device_count(C.byref(n))
    if st != SK_OK:
        return 0
    return n.value


def stream(device: int) -> int:
    s = _streams.get(device)
    if s is None:
        out = C.c_size_t(0)
        call("sk_stream_default", device, C.byref(out))
        s = _streams[device] = out.value
    return s


def sync(device: int) -> None:
    call("sk_stream_sync", stream(device))


def malloc(device: int, nbytes: int) -> int:
    out = C.c_void_p(0)
    call("sk_malloc", device, nbytes, C.byref(out))
    return out.value or 0


def free(device: int, ptr: int) -> None:
    call("sk_free", device, ptr)


def malloc_shareable(device: int, nbytes: int) -> int:
    out = C.c_void_p(0)
    call("sk_malloc_shareable", device, nbytes, C.byref(out))
    return out.value or 0


def free_shareable(device: int, ptr: int) -> None:
    call("sk_free_shareable", device, ptr)


def host_alloc_pinned(nbytes: int) -> int:
    out = C.c_void_p(0)
    call("sk_host_alloc_pinned", nbytes, C.byref(out))
    return out.value or 0


def host_free_pinned(ptr: int) -> None:
    call("sk_host_free_pinned", ptr)


def memcpy(dst: int, src: int, nbytes: int, device: int) -> None:
    call("sk_memcpy_async", dst, src, nbytes, stream(device))


def memmove(dst: int, src: int, nbytes: int, device: int) -> None:
    call("sk_memmove_async", dst, src, nbytes, stream(device))


def memset(dst: int, byte: int, nbytes: int, device: int) -> None:
    call("sk_memset_async", dst, byte, nbytes, stream(device))


class Event:
    """CUDA event on the library's streams (device-side timing)."""

    def __init__(self) -> None:
        out = C.c_size_t(0)
        call("sk_event_create", C.byref(out))
        self.handle = out.value

    def record(self, device: int) -> None:
        call("sk_event_record", self.handle, stream(device))

    def elapsed_ms(self, later: "Event") -> float:
        ms = C.c_float(0.0)
        call("sk_event_elapsed_ms", self.handle, later.handle, C.byref(ms))
        return float(ms.value)

    def __del__(self) -> None:  # pragma: no cover - interpreter teardown order
        try:
            if _lib is not None and self.handle:
                _lib.sk_event_destroy(self.handle)
        except Exception:
            pass
