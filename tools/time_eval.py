"""Event-timed eca_area_hausdorff over 256 (pred, truth) 1080p pairs: truth =
renderer circles of the C2 mix, pred = truth perturbed by ~1 px (a typical fit)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2210_14771_b200 import _lib, api, metrics  # noqa: E402
from support import synth  # noqa: E402

B, W, H = 256, 1920, 1080
dev = torch.device('cuda', 0)
specs = synth.bench_specs(40, W, H, seed=2024)
rng = np.random.default_rng(0)
truth = [specs[i % 40][1].circle for i in range(B)]
pred = [None if t is None else type(t)(t.cx + rng.normal(0, 1), t.cy + rng.normal(0, 1), t.r + rng.normal(0, 1))
        for t in truth]
rp, rt = api._area_records(pred, dev), api._area_records(truth, dev)
dims = torch.tensor([[W, H]] * B, dtype=torch.int32, device=dev)
lib = _lib.load()
nb = ctypes.c_int64()
_lib.check(lib.eca_nh_workspace_bytes(B, W, H, 1.0, ctypes.byref(nb)), "ws")
ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
hd = torch.empty(B, dtype=torch.float64, device=dev)
st = torch.empty(B, dtype=torch.int32, device=dev)
s = api._stream(dev)


def launch():
    _lib.check(lib.eca_area_hausdorff(api._ptr(rp), api._ptr(rt), api._ptr(dims), B, W, H, 1.0, api._ptr(ws),
                                      nb.value, api._ptr(hd), api._ptr(st), s), "hd")


for _ in range(3):
    launch()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    launch()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
print(f"{B} samples: {ms * 1e3:.1f} us/launch = {B / ms * 1e3:.0f} samples/s; mean NH "
      f"{float((hd.cpu().numpy() * metrics.REF_DIAGONAL / np.hypot(W, H)).mean()):.4f}")
