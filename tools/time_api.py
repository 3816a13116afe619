"""Wall-clock latency of the public single-frame API (C1 1080p frame):
estimate(cuda tensor) and estimate(numpy), p50 / p99 over 1000 calls."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb  # noqa: E402
from support import synth  # noqa: E402

frame = synth.c1_frame()
t = torch.from_numpy(frame).cuda()
for name, src in (("cuda", t), ("numpy", frame)):
    for _ in range(50):
        eb.estimate(src)
    ts = []
    for _ in range(1000):
        w = time.perf_counter()
        eb.estimate(src)
        ts.append((time.perf_counter() - w) * 1e3)
    print(f"estimate({name}) p50 {np.percentile(ts, 50):.4f} ms  p99 {np.percentile(ts, 99):.4f} ms")
print(eb.estimate(frame))
