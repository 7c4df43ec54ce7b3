"""How often does Python's `d ** 2` (glibc pow) instead of `d * d` change a
particle's float32 variance? (reconstruct.py:109-110 squares with `** 2`; the
GPU kernel multiplies.) Runs the reference reconstruction's variance sums
both ways over generated events and counts differing f32 results.

usage: PYTHONPATH=/root/reference/pkg/src python tools/pow_check.py [events] [w] [h]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import restate as R  # noqa: E402


def variances(energy, noise, w, h):
    """(vx, vy) per particle, each computed with ** 2 and with x * x (restate.reconstruct's walk)."""
    out = []
    ratio = (energy / noise).astype(np.float32)
    n = w * h
    cand = np.flatnonzero(ratio > np.float32(5.0))
    seeds = cand[np.argsort(-energy[cand], kind="stable")]
    consumed = np.zeros(n, bool)
    for s in seeds:
        s = int(s)
        if consumed[s]:
            continue
        sy, sx = divmod(s, w)
        contrib = []
        for y in range(max(0, sy - 2), min(h - 1, sy + 2) + 1):
            for x in range(max(0, sx - 2), min(w - 1, sx + 2) + 1):
                f = y * w + x
                if not consumed[f] and ratio[f] > np.float32(2.0):
                    consumed[f] = True
                    contrib.append(f)
        sw = swx = swy = 0.0
        for f in contrib:
            e = float(energy[f])
            sw += e
            swx += e * (f % w)
            swy += e * (f // w)
        xbar, ybar = swx / sw, swy / sw
        res = []
        for sq in (lambda d: d ** 2, lambda d: d * d):
            vx = vy = 0.0
            for f in contrib:
                e = float(energy[f])
                vx += e * sq(f % w - xbar)
                vy += e * sq(f // w - ybar)
            res.append((np.float32(vx / sw), np.float32(vy / sw), vx, vy))
        out.append(res)
    return out


if __name__ == "__main__":
    events = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    w = int(sys.argv[2]) if len(sys.argv) > 2 else 436
    h = int(sys.argv[3]) if len(sys.argv) > 3 else 436
    parts = f32_diff = f64_diff = 0
    for seed in range(events):
        ev = R.generate_event(w, h, seed=1000 + seed, density=0.002)
        e = R.calibrate(ev["counts"], ev["parameter_A"], ev["parameter_B"])
        nz = R.noise(e, ev["noise_A"], ev["noise_B"], ev["noisy"])
        for (px, py, dx, dy), (mx, my, ex, ey) in variances(e, nz, w, h):
            parts += 1
            f64_diff += (dx != ex) + (dy != ey)
            f32_diff += (px.tobytes() != mx.tobytes()) + (py.tobytes() != my.tobytes())
    print(f"events={events} grid={w}x{h} particles={parts} variances={2 * parts} "
          f"f64 sums differing={f64_diff} f32 variances differing={f32_diff}")
