import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.profile_one import job
from paper_2511_04853_b200 import _native as nat
fn = job("jagged")
for _ in range(3): fn()
nat.sync(0)
a, b = nat.Event(), nat.Event()
a.record(0); t0 = time.perf_counter()
for _ in range(20): fn()
b.record(0); nat.sync(0); t1 = time.perf_counter()
print(f"pack: {a.elapsed_ms(b)/20*1e3:.1f} us/call (events), {1e6*(t1-t0)/20:.1f} us/call (wall)")
