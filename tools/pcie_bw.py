"""Pinned host <-> device copy bandwidth (the e2e path's ceiling), CUDA events."""
import torch
for mb in (21, 210):
    n = mb * 1_000_000
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        print(f"{name} {mb} MB: {ms:.3f} ms = {n / ms / 1e6:.1f} GB/s")
