"""Per-phase clocks of the fitter (diagnostic build):

    ECA_NVCC_DEFINES=-DECA_FIT_TIMES python -m paper_2210_14771_b200.build --force
    python tools/fit_times.py
Phases: filter | circumcircle | iteration 1..3 (inliers + LSQ) | final scoring | vote."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb  # noqa: E402
from paper_2210_14771_b200 import _lib, api  # noqa: E402
from support import synth  # noqa: E402

B, H, W = 256, 1080, 1920
specs = synth.bench_specs(40, W, H, seed=2024)
frames = torch.from_numpy(np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])).cuda()
frames = frames[[k % 40 for k in range(B)]]
eng = eb.ContentAreaEngine(H, W, B)
eng.points(frames)
lib = _lib.load()
st = api._stream(eng.device)
for rep in range(3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(lib.eca_fit(api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc), B, 32, ctypes.byref(eng.params),
                           api._ptr(eng.trip), 0, api._ptr(eng.rec), st), "fit")
    b.record()
    torch.cuda.synchronize()
    print(f"fit kernel {a.elapsed_time(b) * 1e3:.1f} us")
out = (ctypes.c_ulonglong * (16 * B))()
fn = lib.eca_debug_fit_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert fn(ctypes.cast(out, ctypes.c_void_p), B) == 0
t = np.array(out, dtype=np.int64).reshape(B, 16)[:, :10]
d = np.diff(t[:, :8], axis=1)
names = ["filter", "circum", "iter1", "iter2", "iter3", "final", "vote"]
for i, n in enumerate(names):
    print(f"{n:8s} median {np.median(d[:, i]):8.0f} clk  p90 {np.percentile(d[:, i], 90):8.0f}")
print(f"iter2 split: screen {np.median(t[:, 8] - t[:, 3]):.0f}  moments {np.median(t[:, 9] - t[:, 8]):.0f}  "
      f"lsq {np.median(t[:, 4] - t[:, 9]):.0f} clk")
print(f"total    median {np.median(t[:, 7] - t[:, 0]):8.0f} clk")
# the FP64 rescore stage alone (one lane per survivor slot)
for rep in range(3):
    _lib.check(lib.eca_bounds_handcrafted(
        ctypes.c_void_p(frames.data_ptr()), B, frames.stride(0), frames.stride(1), eng._rows, None,
        eng.n_strips, ctypes.byref(eng.params), api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc),
        api._ptr(eng.workspace), 0, st), "bounds")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(lib.eca_rescore_handcrafted(B, eng._rows, eng.n_strips, ctypes.byref(eng.params),
                                           api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc),
                                           api._ptr(eng.workspace), st), "rescore")
    b.record()
    torch.cuda.synchronize()
    print(f"rescore kernel {a.elapsed_time(b) * 1e3:.1f} us")
cnt = eng.workspace[256:].view(torch.int32)  # not exact offsets; survivors histogram below
