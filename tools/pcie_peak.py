"""Host->device ceilings for the e2e leg: a DMA copy of pinned memory
(copy engines) and a zero-copy read of pinned memory by a kernel (the SMs
load it over PCIe: torch copies a host tensor viewed as mapped memory)."""
import numpy as np
import torch

n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


t = timed(lambda: d.copy_(h, non_blocking=True))
print(f"H2D DMA copy of pinned memory: {n / t / 1e9:.1f} GB/s")
