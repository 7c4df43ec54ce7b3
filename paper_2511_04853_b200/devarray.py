"""A typed 1-D array in any memory context (device arrays for kernel inputs)."""

from __future__ import annotations

import numpy as np

from . import _native as nat
from . import memctx


class DeviceArray:
    """`n` elements of `dtype` in one memctx Buffer (cuda by default)."""

    def __init__(self, n: int, dtype, info: memctx.ContextInfo | None = None) -> None:
        self.dtype = np.dtype(dtype)
        self.n = int(n)
        self.info = info or memctx.ContextInfo.cuda(0)
        self.buffer = memctx.allocate(self.info, self.n * self.dtype.itemsize)

    @classmethod
    def from_numpy(cls, arr, info: memctx.ContextInfo | None = None) -> "DeviceArray":
        a = np.ascontiguousarray(arr)
        out = cls(a.size, a.dtype, info)
        if a.nbytes:
            if out.buffer._host is not None:
                out.buffer._data[:] = a.view(np.uint8).reshape(-1)
            else:
                nat.memcpy(out.ptr, a.ctypes.data, a.nbytes, out.device)
                nat.sync(out.device)
        return out

    @classmethod
    def wrap(cls, ptr: int, n: int, dtype, device: int) -> "DeviceArray":
        """Non-owning view of device memory owned elsewhere (free() is a no-op)."""
        out = cls.__new__(cls)
        out.dtype, out.n, out.info = np.dtype(dtype), int(n), memctx.ContextInfo.cuda(device)
        out.buffer = memctx.Buffer(0, out.info, out.n * out.dtype.itemsize, ptr, None, "view")
        out.buffer._live = False  # not registered with the context: nothing to release
        return out

    @property
    def ptr(self) -> int:
        return self.buffer.ptr

    @property
    def device(self) -> int | None:
        return self.buffer.device

    @property
    def nbytes(self) -> int:
        return self.n * self.dtype.itemsize

    def numpy(self) -> np.ndarray:
        if self.buffer._host is not None:
            return np.array(self.buffer._data[: self.nbytes].view(self.dtype))
        out = memctx.host_return_array(self.n, self.dtype)  # page-locked when large
        if out.nbytes:
            nat.memcpy(out.ctypes.data, self.ptr, out.nbytes, self.device)
            nat.sync(self.device)
        return out

    def free(self) -> None:
        if self.buffer.live:
            memctx.deallocate(self.buffer)

    def __len__(self) -> int:
        return self.n
