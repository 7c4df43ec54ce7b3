"""Numpy restatement of the reference hot path (oracle; see oracle/__init__.py)."""

from __future__ import annotations

import numpy as np

# ---- byte geometry -----------------------------------------------------------------------

_CODES = {"bool": "?", "u8": "u1", "u16": "<u2", "u32": "<u4", "u64": "<u8", "i32": "<i4", "i64": "<i8",
          "f32": "<f4", "f64": "<f8"}


def packed_dtype(fields: list[tuple[str, str, int]]) -> np.dtype:
    """Packed AoS record of main-tag element leaves in plan order, multi-slot
    leaves inline as (extent,) sub-arrays, no padding (layouts.py:575-585)."""
    out = []
    for name, code, extent in fields:
        out.append((name, _CODES[code], (extent,)) if extent > 1 else (name, _CODES[code]))
    return np.dtype(out)


# ---- K1 / K2: per-leaf conversion (transfer.py:196-233) -----------------------------------

def aos_to_planes(records: np.ndarray) -> dict[str, list[np.ndarray]]:
    """AoS struct array -> {leaf: [plane per slot]} contiguous planes.
    Restates transfer.py:203-205 (column view, slot k) + 226 (ascontiguousarray)."""
    out = {}
    for name in records.dtype.names:
        col = records[name]
        if col.ndim == 1:
            out[name] = [np.ascontiguousarray(col)]
        else:
            out[name] = [np.ascontiguousarray(col[:, k]) for k in range(col.shape[1])]
    return out


def planes_to_aos(planes: dict[str, list[np.ndarray]], dtype: np.dtype, n: int) -> np.ndarray:
    """Planes -> packed AoS records. Restates transfer.py:206-220 (dcol[...] = plane)."""
    rec = np.zeros(n, dtype)
    for name in dtype.names:
        col = rec[name]
        for k, plane in enumerate(planes[name]):
            if col.ndim == 1:
                col[...] = plane[:n]
            else:
                col[:, k] = plane[:n]
    return rec


# ---- K3: AoSoA with subset/reorder/cast (no reference path) --------

def to_aosoa(records: np.ndarray, fields: list[tuple[str, str]], lanes: int, tile_bytes: int | None = None) -> bytes:
    """Tiles of `lanes` records; per tile one block of `lanes` elements per
    selected field (in the requested order) cast with numpy astype; lanes past
    n and tile padding are zero."""
    n = records.size
    ntiles = -(-n // lanes)
    sizes = [np.dtype(_CODES[c]).itemsize for _, c in fields]
    body = sum(lanes * s for s in sizes)
    tile_bytes = tile_bytes or -(-body // 16) * 16
    out = np.zeros(ntiles * tile_bytes, dtype=np.uint8)
    off = 0
    for (name, code), sz in zip(fields, sizes):
        vals = np.zeros(ntiles * lanes, dtype=_CODES[code])
        with np.errstate(over="ignore", invalid="ignore"):  # numpy's own cast of random bit patterns
            vals[:n] = records[name].astype(_CODES[code])
        blocks = vals.view(np.uint8).reshape(ntiles, lanes * sz)
        out.reshape(ntiles, tile_bytes)[:, off : off + lanes * sz] = blocks
        off += lanes * sz
    return out.tobytes()


# ---- K4: jagged packing (collection.py:537-556, transfer.py:297-320) ----------------------

def jagged_pack(lens: np.ndarray, offsets: np.ndarray, pool: np.ndarray, index_dtype) -> tuple[np.ndarray, np.ndarray]:
    """prefix = [0, cumsum(int64(lens))].astype(index dtype) (collection.py:552-554);
    packed pool = concatenation of the segments in record order (collection.py:546, 555-556)."""
    lens = np.asarray(lens, dtype=np.int64)
    prefix = np.zeros(lens.size + 1, dtype=index_dtype)
    if lens.size:
        prefix[1:] = np.cumsum(lens).astype(index_dtype)
    segs = [pool[o : o + l] for o, l in zip(np.asarray(offsets, np.int64), lens)]
    packed = np.concatenate(segs) if segs else pool[:0]
    return prefix, packed


# ---- K5: the case-study kernel (detector/schemas.py:29-41) -------------------------------

def calibrate(counts: np.ndarray, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """energy = A * counts.astype(f32) + B (detector/schemas.py:33)."""
    return a * counts.astype(np.float32) + b


def noise(energy: np.ndarray, na: np.ndarray, nb: np.ndarray, noisy: np.ndarray) -> np.ndarray:
    """nA * sqrt(max(E, 0)) + nB, doubled where noisy (detector/schemas.py:37-41)."""
    e = np.maximum(energy, np.float32(0.0))
    n = na * np.sqrt(e) + nb
    return np.where(noisy, n * np.float32(2.0), n)


# ---- inputs: splitmix64 events (detector/events.py:37-133) -------------------------------

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)
_FOOT = [[np.exp(-(dx * dx + dy * dy) / 2.88) for dx in range(-2, 3)] for dy in range(-2, 3)]


def mix_stream(seed: int, start: int, count: int) -> np.ndarray:
    """splitmix64 outputs [start, start+count) (events.py:37-44)."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        return z ^ (z >> np.uint64(31))


def generate_event(w: int, h: int, seed: int = 0, density: float = 0.0) -> dict[str, np.ndarray]:
    """Sensor input columns of one event (events.py:85-133)."""
    n = w * h
    pu = (mix_stream(seed, 0, 16) >> np.uint64(11)) * (2.0 ** -53)
    a = np.array([0.3 + 0.7 * pu[4 * t] for t in range(4)], dtype=np.float32)
    b = np.array([2.0 * pu[4 * t + 1] for t in range(4)], dtype=np.float32)
    na = np.array([1.0 + 1.0 * pu[4 * t + 2] for t in range(4)], dtype=np.float32)
    nb = np.array([0.5 + 1.5 * pu[4 * t + 3] for t in range(4)], dtype=np.float32)
    so = mix_stream(seed, 16, 3 * n).reshape(n, 3)
    stype = (so[:, 0] & np.uint64(3)).astype(np.uint8)
    counts = (so[:, 1] & np.uint64(15)).astype(np.uint64)
    noisy = (so[:, 2] % np.uint64(50)) == 0
    n_dep = int(round(density * n))
    if n_dep:
        do = mix_stream(seed, 16 + 3 * n, 3 * n_dep).reshape(n_dep, 3)
        for d in range(n_dep):
            cx, cy = int(do[d, 0] % np.uint64(w)), int(do[d, 1] % np.uint64(h))
            amp = 500 + int(do[d, 2] % np.uint64(1500))
            for dy in range(-2, 3):
                y = cy + dy
                if 0 <= y < h:
                    for dx in range(-2, 3):
                        x = cx + dx
                        if 0 <= x < w:
                            counts[y * w + x] += int(amp * _FOOT[dy + 2][dx + 2])
    return {"type": stype, "counts": counts, "noisy": noisy, "parameter_A": a[stype], "parameter_B": b[stype],
            "noise_A": na[stype], "noise_B": nb[stype]}


SENSOR_AOS_DTYPE = np.dtype([
    ("type", "u1"), ("counts", "<u8"), ("energy", "<f4"),
    ("calibration_data", [("noisy", "?"), ("parameter_A", "<f4"), ("parameter_B", "<f4"),
                          ("noise_A", "<f4"), ("noise_B", "<f4")]),
])


def sensor_aos(ev: dict[str, np.ndarray]) -> np.ndarray:
    """HandwrittenAosPipeline.fill (detector/baselines.py:133-146): energy = 0."""
    s = np.empty(ev["type"].size, SENSOR_AOS_DTYPE)
    s["type"], s["counts"], s["energy"] = ev["type"], ev["counts"], 0
    cal = s["calibration_data"]
    for k in ("noisy", "parameter_A", "parameter_B", "noise_A", "noise_B"):
        cal[k] = ev[k]
    return s


# ---- particle reconstruction (detector/reconstruct.py:53-136) -----------------------------

def reconstruct(energy, noise, sensor_type, noisy, width: int, height: int) -> dict:
    """Greedy seeded 5x5 clustering, restated from reconstruct.py:53-136: seeds
    (ratio > 5) in descending energy / ascending index; each unconsumed seed
    takes the unconsumed ratio > 2 cells of its grid-clipped window in
    row-major order; per-type f64 sums rounded once to f32; energy-weighted
    f64 centroid and two-pass variance."""
    n = width * height
    energy = np.asarray(energy, dtype=np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = energy / np.asarray(noise, dtype=np.float32)
    cand = np.flatnonzero(ratio > np.float32(5.0))
    seeds = cand[np.argsort(-energy[cand], kind="stable")]
    consumed = np.zeros(n, dtype=bool)
    out = {k: [] for k in ("energy", "x", "y", "origin", "x_variance", "y_variance", "significance",
                           "E_contribution", "noisy_count", "sensors")}
    for s in seeds:
        s = int(s)
        if consumed[s]:
            continue
        sy, sx = divmod(s, width)
        contrib = []
        for y in range(max(0, sy - 2), min(height - 1, sy + 2) + 1):
            for x in range(max(0, sx - 2), min(width - 1, sx + 2) + 1):
                f = y * width + x
                if not consumed[f] and ratio[f] > np.float32(2.0):
                    consumed[f] = True
                    contrib.append(f)
        e64, sig64, cnt = [0.0] * 4, [0.0] * 4, [0] * 4
        sw = swx = swy = 0.0
        for f in contrib:
            e, t = float(energy[f]), int(sensor_type[f])
            e64[t] += e
            sig64[t] += float(ratio[f])
            cnt[t] += bool(noisy[f])
            sw += e
            swx += e * (f % width)
            swy += e * (f // width)
        xbar, ybar = swx / sw, swy / sw
        vx = vy = 0.0
        for f in contrib:
            e = float(energy[f])
            vx += e * (f % width - xbar) ** 2
            vy += e * (f // width - ybar) ** 2
        e32 = [np.float32(v) for v in e64]
        out["energy"].append(np.float32(float(e32[0]) + float(e32[1]) + float(e32[2]) + float(e32[3])))
        out["x"].append(np.float32(xbar))
        out["y"].append(np.float32(ybar))
        out["origin"].append(s)
        out["x_variance"].append(np.float32(vx / sw))
        out["y_variance"].append(np.float32(vy / sw))
        out["significance"].append([np.float32(v) for v in sig64])
        out["E_contribution"].append(e32)
        out["noisy_count"].append(cnt)
        out["sensors"].append(np.array(contrib, dtype=np.uint64))
    m = len(out["energy"])
    res = {k: np.array(out[k], dtype=dt) for k, dt in (("energy", np.float32), ("x", np.float32), ("y", np.float32),
                                                       ("origin", np.uint64), ("x_variance", np.float32),
                                                       ("y_variance", np.float32))}
    res["significance"] = np.array(out["significance"], np.float32).reshape(m, 4)
    res["E_contribution"] = np.array(out["E_contribution"], np.float32).reshape(m, 4)
    res["noisy_count"] = np.array(out["noisy_count"], np.uint8).reshape(m, 4)
    res["sensor_lens"] = np.array([a.size for a in out["sensors"]], np.int32)
    res["sensors"] = np.concatenate(out["sensors"]) if m else np.empty(0, np.uint64)
    return res


# ---- bench inputs: the splitmix64 record images sk_fill_random writes --------------------

def splitmix_image(seed: int, first_word: int, byte_off: int, nbytes: int) -> np.ndarray:
    """Bytes [byte_off, byte_off + nbytes) of the synthetic image whose 8-byte
    word w is splitmix64(seed, first_word + w), little-endian (the same
    counter-based mixer as events.py:37-44, keyed by word index). The bench
    uses it to check sampled records of collections too large to copy back."""
    w0, w1 = byte_off // 8, -(-(byte_off + nbytes) // 8)
    words = mix_stream(seed, first_word + w0, w1 - w0)
    raw = words.view(np.uint8)
    s = byte_off - w0 * 8
    return raw[s : s + nbytes]
