"""Host-side cost of the pieces of estimate(cuda tensor) (C1 1080p frame):
median microseconds over 2000 calls of each piece, and of the whole call."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb  # noqa: E402
from paper_2210_14771_b200 import api  # noqa: E402
from support import synth  # noqa: E402

frame = synth.c1_frame()
t = torch.from_numpy(frame).cuda()
eb.estimate(t)
cfg = api.config_default()
key = (1080, 1920, cfg, 0, 0)
est = api._FRAME_ESTIMATORS[key]
stream = torch.cuda.current_stream()


def med(fn, n=2000):
    for _ in range(50):
        fn()
    ts = []
    for _ in range(n):
        w = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - w)
    return 1e6 * float(np.median(ts))


parts = {
    "estimate(cuda) total": lambda: eb.estimate(t),
    "validate_frame": lambda: api.validate_frame(t),
    "config_default": api.config_default,
    "_check_config": lambda: api._check_config(cfg),
    "cache key + dict get": lambda: api._FRAME_ESTIMATORS.get((1080, 1920, cfg, 0, t.device.index)),
    "hash(cfg)": lambda: hash(cfg),
    "torch.cuda.current_device": torch.cuda.current_device,
    "torch.cuda.current_stream(dev)": lambda: torch.cuda.current_stream(est.dev),
    "_run (launch + sync + record)": lambda: est._run(t),
    "stream.synchronize (idle)": stream.synchronize,
    "t.stride/data_ptr": lambda: (t.stride(2), t.stride(1), t.stride(0), t.data_ptr()),
}
for k, f in parts.items():
    print(f"{k:34s} {med(f):7.2f} us")
