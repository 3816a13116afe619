"""ncu target for K5 crop_copy_kernel: 256 x 1080p frames, C2-like crop
rectangles (centred circles, r 400-560 px) packed back to back.
usage: ncu ... -k regex:crop_copy python tools/ncu_crop.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2210_14771_b200 import _lib, api  # noqa: E402

B, H, W = 256, 1080, 1920
dev = torch.device("cuda:0")
rng = np.random.default_rng(3)
f = torch.randint(0, 256, (B, H, W, 3), dtype=torch.uint8, device=dev)
bounds = np.zeros((B, 4), dtype=np.int32)
for b in range(B):
    cx, cy, r = 960 + rng.uniform(-50, 50), 540 + rng.uniform(-30, 30), rng.uniform(400, 560)
    h = r / np.sqrt(2.0)
    bounds[b] = (int(np.ceil(cx - h)), int(np.ceil(cy - h)), int(np.floor(cx + h)), int(np.floor(cy + h)))
sizes = [(r[2] - r[0] + 1) * (r[3] - r[1] + 1) * 3 for r in bounds]
offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
out = torch.empty(int(sum(sizes)), dtype=torch.uint8, device=dev)
bd, od = torch.from_numpy(bounds).to(dev), torch.from_numpy(offs).to(dev)
max_rows = int(max(r[3] - r[1] + 1 for r in bounds))
lib = _lib.load()
for _ in range(3):
    _lib.check(lib.eca_crop_copy(api._ptr(f), B, f.stride(0), f.stride(1), api._ptr(bd), api._ptr(od),
                                 api._ptr(out), max_rows, api._stream(dev)), "crop_copy")
torch.cuda.synchronize()
print("algorithmic bytes per launch", 2 * int(sum(sizes)))
