"""Write-only HBM bandwidth on this GPU, for the mask writer's roofline:
cudaMemsetAsync and a 16-byte-store fill of the mask buffer size (256 x 1080p
bytes = 530.8 MB), event-timed, median of 20."""
import sys

import numpy as np
import torch
from cuda.bindings import runtime as rt

n = 256 * 1080 * 1920
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


t_ms = timed(lambda: rt.cudaMemsetAsync(buf.data_ptr(), 1, n, st.cuda_stream))
t_fill = timed(lambda: buf.fill_(1))
b16 = buf.view(torch.int32)
t_i32 = timed(lambda: b16.fill_(7))
for name, t in (("cudaMemsetAsync", t_ms), ("torch uint8 fill_", t_fill), ("torch int32 fill_", t_i32)):
    print(f"{name:20s} {t * 1e6:8.1f} us  {n / t / 1e9:7.1f} GB/s")
