#!/usr/bin/env python
"""Write-bandwidth ceiling for the dense-report expand: fill / arange of 8 GiB of int64 (CUDA events)."""
import torch
torch.cuda.set_device(0)
n = 1 << 30
x = torch.empty(n, dtype=torch.int64, device="cuda")
for name, fn in (("fill_", lambda: x.fill_(7)), ("arange(out=)", lambda: torch.arange(n, out=x))):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {best:.3f} ms = {8 * n / best / 1e6:.1f} GB/s written")
