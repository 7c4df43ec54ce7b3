"""Obj8 planes -> AoS (K2) and AoS -> planes (K1) device time at 100M objects (cold: 6.4 GB per launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.profile_one import job  # noqa: E402
from paper_2511_04853_b200 import _native as nat  # noqa: E402

for name in ("obj8_p2a", "obj8_a2p"):
    fn = job(name)
    for _ in range(3):
        fn()
    nat.sync(0)
    a, b = nat.Event(), nat.Event()
    a.record(0)
    for _ in range(10):
        fn()
    b.record(0)
    nat.sync(0)
    ms = a.elapsed_ms(b) / 10
    tag = " ".join(f"{v}={os.environ[v]}" for v in ("SK_TILE_BYTES", "SK_STAGES", "SK_CTAS") if v in os.environ)
    print(f"{name}: {ms:.3f} ms  {6.4e9 / ms / 1e6:.0f} GB/s  frac {6.4e9 / ms / 1e6 / 6546.9:.3f} {tag}", flush=True)
