"""C-ABI failure modes: every bad descriptor is refused with the mapped
exception before any kernel runs (OOM -> AllocationError, bad
range -> CopyError, unsupported -> UnsupportedTransferError)."""

import ctypes as C

import numpy as np
import pytest

import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat
from paper_2511_04853_b200.devarray import DeviceArray

pytestmark = pytest.mark.gpu


def _desc(n=100, nfields=1, src_kind=nat.KIND_AOS, dst_kind=nat.KIND_PLANES, stride=8):
    src = DeviceArray(max(n, 1) * 64, np.uint8)
    dst = DeviceArray(max(n, 1) * 64, np.uint8)
    d = nat.ConvDesc()
    d.n, d.src_kind, d.dst_kind = n, src_kind, dst_kind
    d.src, d.dst = src.ptr, dst.ptr
    d.src_stride, d.dst_stride = stride, stride
    d.nfields = nfields
    for i in range(nfields):
        f = d.fields[i]
        f.src_type = f.dst_type = nat.TYPE_CODES["u32"]
        f.src_off = f.dst_off = 4 * i
        f.src_plane = src.ptr
        f.dst_plane = dst.ptr + 4096 * i
    return d, (src, dst)


def _run(d):
    nat.call("sk_convert", C.byref(d), 0, nat.stream(0))
    nat.sync(0)


def test_field_outside_record_is_a_copy_error():
    d, keep = _desc()
    d.fields[0].src_off = 6  # 4 bytes at 6 in an 8-byte record
    with pytest.raises(sk.CopyError):
        _run(d)


def test_float_to_int_cast_is_unsupported():
    d, keep = _desc()
    d.fields[0].src_type = nat.TYPE_CODES["f32"]
    d.fields[0].dst_type = nat.TYPE_CODES["i32"]
    with pytest.raises(sk.UnsupportedTransferError):
        _run(d)


def test_overlapping_destination_fields_are_refused():
    d, keep = _desc(nfields=2, dst_kind=nat.KIND_AOS, src_kind=nat.KIND_PLANES)
    d.fields[1].dst_off = 2
    with pytest.raises(sk.SoakitError):
        _run(d)


@pytest.mark.parametrize("bad", [dict(nfields=0), dict(nfields=65), dict(n=-1)])
def test_bad_counts(bad):
    d, keep = _desc(nfields=min(max(bad.get("nfields", 1), 1), 64), n=max(bad.get("n", 100), 0))
    if "nfields" in bad:
        d.nfields = bad["nfields"]
    if "n" in bad:
        d.n = bad["n"]
    with pytest.raises(sk.SoakitError):
        _run(d)


def test_bad_aosoa_lanes():
    d, keep = _desc(dst_kind=nat.KIND_AOSOA, stride=4096)
    d.dst_lanes = 3
    with pytest.raises(sk.SoakitError):
        _run(d)


def test_zero_records_is_a_no_op():
    d, keep = _desc(n=0)
    _run(d)


def test_device_oom_is_allocation_error():
    with pytest.raises(sk.AllocationError):
        nat.malloc(0, 1 << 50)  # 1 PiB
    nat.sync(0)  # the stream stays usable
    DeviceArray(16, np.uint8).free()
