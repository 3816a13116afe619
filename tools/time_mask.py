"""Time K4 draw_mask (256 x 1080p, accepted circles of varied size) against a
torch fill of the same buffer (the write-only ceiling).  usage: python tools/time_mask.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2210_14771_b200 import _lib, api

B, H, W = 256, 1080, 1920
dev = torch.device("cuda:0")
rng = np.random.default_rng(1)
rec = np.zeros(B, dtype=[("cx", "f8"), ("cy", "f8"), ("r", "f8"), ("score", "f8"), ("inl", "i4"), ("st", "i4")])
rec["cx"] = 960 + rng.uniform(-40, 40, B)
rec["cy"] = 540 + rng.uniform(-40, 40, B)
rec["r"] = rng.uniform(400, 1100, B)
rd = torch.from_numpy(rec.view(np.uint8).copy()).to(dev)
out = torch.empty((B, H, W), dtype=torch.uint8, device=dev)
lib = _lib.load()
st = api._stream(dev)


def timeit(fn, steps=30):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def mask():
    _lib.check(lib.eca_draw_mask(api._ptr(rd), B, H, W, api._ptr(out), H * W, st), "mask")


ms = timeit(mask)
mf = timeit(lambda: out.fill_(1))
n = B * H * W
print(f"mask {ms*1e3:.1f} us {n/ms/1e6:.0f} GB/s | torch fill {mf*1e3:.1f} us {n/mf/1e6:.0f} GB/s")
