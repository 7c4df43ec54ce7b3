"""Schemas and seeded synthetic inputs for the BASELINE.json configurations.

  OBJ8     config 1/5: f0..f7 alternating f32 (even) / i32 (odd), 32-byte AoS
  SENSOR   config 2:   sensor.SENSOR_SCHEMA, 30-byte AoS, events of W x H cells
  CLUSTER  config 3:   records with a jagged u64 member list (i32 index)
  CLUSTER2 config 3b:  jagged members {adc i32, t f32} -> two pools
  TRACK    config 4:   x,y,z,px,py,pz f64; charge i32; id u64 -> 60-byte AoS

Generators are plain numpy (input synthesis, not the measured path). Large
device-resident inputs are synthesised on the GPU with sk_fill_random.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from . import schema as sc

OBJ8_SCHEMA = sc.Schema("Obj8", tuple(
    sc.declare_per_item(f"f{i}", sc.F32 if i % 2 == 0 else sc.I32) for i in range(8)))

TRACK_SCHEMA = sc.Schema("Track", (
    sc.declare_per_item("x", sc.F64), sc.declare_per_item("y", sc.F64), sc.declare_per_item("z", sc.F64),
    sc.declare_per_item("px", sc.F64), sc.declare_per_item("py", sc.F64), sc.declare_per_item("pz", sc.F64),
    sc.declare_per_item("charge", sc.I32), sc.declare_per_item("id", sc.U64),
))

CLUSTER_SCHEMA = sc.Schema("Cluster", (
    sc.declare_per_item("seed", sc.U64),
    sc.declare_jagged("members", sc.I32, sc.U64),
))

CLUSTER2_SCHEMA = sc.Schema("Cluster2", (
    sc.declare_per_item("seed", sc.U64),
    sc.declare_jagged("hits", sc.I32, [sc.declare_per_item("adc", sc.I32), sc.declare_per_item("t", sc.F32)]),
))

OBJ8_AOS_DTYPE = np.dtype([(f"f{i}", "<f4" if i % 2 == 0 else "<i4") for i in range(8)])
TRACK_AOS_DTYPE = np.dtype([("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("px", "<f8"), ("py", "<f8"),
                            ("pz", "<f8"), ("charge", "<i4"), ("id", "<u8")])
HIT_DTYPE = np.dtype([("adc", "<i4"), ("t", "<f4")])


def obj8_records(n: int, seed: int = 1234) -> np.ndarray:
    """Config-1 inputs: f32 ~ N(0,1) with 1% special values (signed zeros, infs,
    subnormals, NaNs with payloads), i32 uniform over the full range."""
    rng = np.random.default_rng(seed)
    rec = np.empty(n, OBJ8_AOS_DTYPE)
    specials = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x00000001, 0x807FFFFF,
                         0x7FC00001, 0x7F800ABC, 0xFFC12345, 0x7FBFFFFF], dtype=np.uint32)
    for i in range(8):
        name = f"f{i}"
        if i % 2 == 0:
            v = rng.standard_normal(n).astype(np.float32)
            bits = v.view(np.uint32)
            hit = rng.random(n) < 0.01
            bits[hit] = specials[rng.integers(0, specials.size, int(hit.sum()))]
            rec[name] = bits.view(np.float32)
        else:
            rec[name] = rng.integers(-(1 << 31), 1 << 31, n, dtype=np.int64).astype(np.int32)
    return rec


def track_records(n: int, seed: int = 42) -> np.ndarray:
    """Config-4 inputs: f64 ~ 1e3 * N(0,1) plus cast edge cases (f32 overflow,
    subnormal results, exact RNE ties, NaN payloads)."""
    rng = np.random.default_rng(seed)
    rec = np.empty(n, TRACK_AOS_DTYPE)
    edges = np.array([3.5e38, -3.5e38, 1e-45, 7e-46, 1.5e-45, 1.0 + 2.0 ** -24, 1.0 + 3 * 2.0 ** -24,
                      np.inf, -np.inf, 0.0, -0.0, 2.0 ** -149, 2.0 ** -150], dtype=np.float64)
    nans = np.array([0x7FF8DEAD00000000, 0xFFF0000000000001, 0x7FF4000000000000, 0x7FFFFFFFFFFFFFFF],
                    dtype=np.uint64).view(np.float64)
    for name in ("x", "y", "z", "px", "py", "pz"):
        v = rng.standard_normal(n) * 1e3
        hit = rng.random(n) < 0.01
        pool = np.concatenate([edges, nans])
        v[hit] = pool[rng.integers(0, pool.size, int(hit.sum()))]
        rec[name] = v
    rec["charge"] = rng.integers(-(1 << 31), 1 << 31, n, dtype=np.int64).astype(np.int32)
    rec["id"] = rng.integers(0, np.iinfo(np.uint64).max, n, dtype=np.uint64, endpoint=True)
    return rec


def cluster_inputs(n: int, seed: int = 7, max_len: int = 20, member_dtype=np.uint64):
    """Config-3 inputs: lens ~ U[0, max_len], segments scattered through a source
    pool in shuffled record order with random slack between them."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len + 1, n).astype(np.int32)
    order = rng.permutation(n)
    slack = rng.integers(0, 4, n)
    offsets = np.empty(n, dtype=np.int64)
    for_order = lens[order].astype(np.int64) + slack
    starts = np.concatenate([[0], np.cumsum(for_order)[:-1]]) if n else np.empty(0, np.int64)
    offsets[order] = starts
    pool_len = int(for_order.sum()) if n else 0
    if np.dtype(member_dtype) == HIT_DTYPE:
        pool = np.empty(pool_len, HIT_DTYPE)
        pool["adc"] = rng.integers(-(1 << 31), 1 << 31, pool_len, dtype=np.int64).astype(np.int32)
        pool["t"] = rng.standard_normal(pool_len).astype(np.float32)
    else:
        pool = rng.integers(0, np.iinfo(np.uint64).max, pool_len, dtype=np.uint64, endpoint=True)
    return lens, offsets, pool


def fill_random_device(ptr: int, nbytes: int, seed: int, device: int, first_word: int = 0) -> None:
    """splitmix64 bits; a shard at byte offset 8*first_word of the global image
    gets exactly its slice."""
    nat.call("sk_fill_random", ptr, nbytes, seed, first_word, nat.stream(device))
