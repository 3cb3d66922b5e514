"""Pinned host->device copy rate with one, two and four concurrent streams (and with a
device->host copy running at the same time)."""
import torch
n = 1 << 27  # 1 GiB of fp64
h = [torch.empty(n // 4, dtype=torch.float64).pin_memory() for _ in range(4)]
d = [torch.empty(n // 4, dtype=torch.float64, device="cuda") for _ in range(4)]
hb = torch.empty(n // 4, dtype=torch.float64).pin_memory()
db = torch.empty(n // 4, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(5)]
for k in (1, 2, 4):
    for with_d2h in (False, True):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r in range(3):
            for i in range(4):
                with torch.cuda.stream(streams[i % k]):
                    d[i].copy_(h[i], non_blocking=True)
            if with_d2h:
                with torch.cuda.stream(streams[4]):
                    hb.copy_(db, non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if False else None
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"streams={k} d2h={with_d2h}: H2D {3 * n * 8 / ms / 1e6:.1f} GB/s", flush=True)
