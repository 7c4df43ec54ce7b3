"""GPU-test helpers: build collections from raw images, read planes back, wrap
device pointers for torch-side verification."""

import numpy as np

import paper_2511_04853_b200 as sk
from paper_2511_04853_b200 import _native as nat
from paper_2511_04853_b200 import layouts as ly
from paper_2511_04853_b200 import memctx as mc
from paper_2511_04853_b200 import transfer as tr

HOST = mc.ContextInfo.host()
PINNED = mc.ContextInfo.pinned()
CUDA = mc.ContextInfo.cuda(0)


def aos_collection(schema, raw: np.ndarray, n: int, info=HOST):
    """AoS collection whose struct image is `raw` (host or pinned)."""
    c = sk.Collection(schema, ly.AOS, info)
    c.resize(n)
    stride = c.layout.record_stride
    c.layout._struct_buf._data[: n * stride] = np.frombuffer(np.ascontiguousarray(raw).tobytes(), np.uint8)[: n * stride]
    return c


def to_host_planes(coll) -> dict:
    """Every plane of every leaf (leaf#k -> bytes) via a host per_field copy."""
    h = sk.Collection(coll.schema, ly.PER_FIELD, HOST)
    tr.copy_collection(h, coll)
    lay = h.layout
    return {f"{lf.dotted}#{k}": np.array(lay._plane_view(lf, k)).view(np.uint8).tobytes()
            for lf in h.plan.leaves for k in range(lay.plane_count(lf))}


def to_host_aos(coll) -> np.ndarray:
    h = sk.Collection(coll.schema, ly.AOS, HOST)
    tr.copy_collection(h, coll)
    n, s = h.size(), h.layout.record_stride
    return np.array(h.layout._struct_buf._data[: n * s])


class CudaView:
    """__cuda_array_interface__ over raw device bytes (torch.as_tensor wraps it)."""

    def __init__(self, ptr: int, nbytes: int) -> None:
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                         "strides": None}


def device_bytes_equal(p1: int, p2: int, nbytes: int, device: int = 0) -> bool:
    import torch

    nat.sync(device)
    a = torch.as_tensor(CudaView(p1, nbytes), device=f"cuda:{device}")
    b = torch.as_tensor(CudaView(p2, nbytes), device=f"cuda:{device}")
    return bool(torch.equal(a, b))


def device_to_numpy(ptr: int, nbytes: int, device: int = 0) -> np.ndarray:
    out = np.empty(nbytes, np.uint8)
    if nbytes:
        nat.memcpy(out.ctypes.data, ptr, nbytes, device)
        nat.sync(device)
    return out
