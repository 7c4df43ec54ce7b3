"""Pinned H2D bandwidth with 1, 2 and 4 concurrent streams (is one DMA engine the limit?)."""
import torch

n = 1 << 30
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    part = n // k
    for _ in range(2):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dev[i * part:(i + 1) * part].copy_(host[i * part:(i + 1) * part], non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    for _ in range(5):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dev[i * part:(i + 1) * part].copy_(host[i * part:(i + 1) * part], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    print(f"streams={k} H2D {5 * n / (a.elapsed_time(b) / 1e3) / 1e9:.1f} GB/s")
