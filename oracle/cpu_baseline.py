"""CPU baseline legs of bench.py (TEST / BASELINE INFRASTRUCTURE ONLY).

The reference's own conversion path, restated on numpy so it runs on the GPU
box without /root/reference: per leaf, a strided column view of the packed
struct, np.ascontiguousarray (the gather) and a byte copy into the plane
(transfer.py:196-228). Timed with the reference protocol: warm-up, then the
mean of the fastest samples (bench.py:214-215).
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os
import time

import numpy as np

OBJ8 = np.dtype([(f"f{i}", "<f4" if i % 2 == 0 else "<i4") for i in range(8)])


def per_leaf_convert(records: np.ndarray, planes: list[np.ndarray]) -> None:
    """transfer.py:203-205 (column), 226 (ascontiguousarray), 228 (copy into plane)."""
    for name, plane in zip(records.dtype.names, planes):
        packed = np.ascontiguousarray(records[name])
        plane.view(np.uint8)[:] = packed.view(np.uint8).reshape(-1)


def mean_of_fastest(samples, keep: int) -> float:
    return sum(sorted(samples)[:keep]) / keep


def single_core(n: int, budget_s: float = 15.0, seed: int = 1) -> dict:
    """Reference path on one core: objects/s and GB/s (64 B/object algorithmic)."""
    rng = np.random.default_rng(seed)
    rec = np.frombuffer(rng.integers(0, 256, n * 32, dtype=np.uint8).tobytes(), OBJ8)
    planes = [np.empty(n, OBJ8[i]) for i in range(8)]
    per_leaf_convert(rec, planes)  # warm-up
    samples = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(samples) < 3:
        t0 = time.perf_counter()
        per_leaf_convert(rec, planes)
        samples.append(time.perf_counter() - t0)
    t = mean_of_fastest(samples, max(1, min(10, len(samples) // 3)))
    return {"seconds": t, "objects_per_s": n / t, "gbs": n * 64 / t / 1e9, "reps": len(samples)}


# ---- multi-core arm ----------------------------------------------------------------------

_G = {}


def _work(span):
    lo, hi = span
    per_leaf_convert(_G["rec"][lo:hi], [pl[lo:hi] for pl in _G["planes"]])
    return hi - lo


def multi_core(n: int, steps: int, warmup: int, procs: int | None = None, seed: int = 1) -> dict:
    """The reference path sharded over all host cores (one process per core).
    Buffers are anonymous shared mappings inherited through fork, so a small
    /dev/shm does not matter."""
    procs = procs or os.cpu_count() or 1
    a = mmap.mmap(-1, n * 32)
    p = mmap.mmap(-1, n * 32)
    try:
        rec = np.frombuffer(a, OBJ8)
        rng = np.random.default_rng(seed)
        chunk = 1 << 24
        for lo in range(0, n * 32, chunk):
            hi = min(lo + chunk, n * 32)
            np.frombuffer(a, np.uint8)[lo:hi] = rng.integers(0, 256, hi - lo, dtype=np.uint8)
        base = np.frombuffer(p, np.uint8)
        _G["rec"] = rec
        _G["planes"] = [base[i * n * 4 : (i + 1) * n * 4].view(OBJ8[i]) for i in range(8)]
        cuts = np.linspace(0, n, procs * 4 + 1).astype(np.int64)
        spans = list(zip(cuts[:-1].tolist(), cuts[1:].tolist()))
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            for _ in range(warmup):
                pool.map(_work, spans)
            times = []
            for _ in range(steps):
                t0 = time.perf_counter()
                done = sum(pool.map(_work, spans))
                times.append(time.perf_counter() - t0)
                assert done == n
        # the children wrote through the shared mapping: spot-check one plane
        assert np.array_equal(_G["planes"][3][: min(n, 1000)], rec["f3"][: min(n, 1000)])
        return {"step_seconds": times, "procs": procs, "n": n}
    finally:
        _G.clear()
        del rec, base
        a.close()
        p.close()
