"""Per-CTA start / end of the streamed step's kernels (diagnostic build):

    ECA_NVCC_DEFINES=-DECA_TIMELINE python -m paper_2210_14771_b200.build --force
    python tools/timeline.py
For a few consecutive steps: each kernel's first start, median start, last
end, relative to the first step's bounds start (us)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb  # noqa: E402
from paper_2210_14771_b200 import _lib  # noqa: E402
from support import synth  # noqa: E402

B, H, W, POOL, NB = 256, 1080, 1920, 2048, 40
specs = synth.bench_specs(NB, W, H, seed=2024)
base = torch.from_numpy(np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])).cuda()
pool = base[[k % NB for k in range(POOL)]].contiguous()
eng = eb.ContentAreaEngine(H, W, B)
n_slots = POOL // B
steps = 40
for i in range(steps):
    eng.run_pipelined(pool[(i % n_slots) * B:(i % n_slots + 1) * B], frames_ready=True)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 64 * 1024 * 2))()
fn = _lib.load().eca_debug_timeline
fn.argtypes = [ctypes.c_void_p]
assert fn(ctypes.cast(buf, ctypes.c_void_p)) == 0
t = np.array(buf, dtype=np.int64).reshape(2, 64, 1024, 2).astype(np.float64)
t0 = None
for seq in range(20, 28):
    for kind, name in ((0, "bounds"), (1, "fit")):
        v = t[kind, seq]
        v = v[(v[:, 0] > 0) & (v[:, 1] > 0)]
        if t0 is None:
            t0 = v[:, 0].min()
        s, e = (v[:, 0] - t0) / 1e3, (v[:, 1] - t0) / 1e3
        dur = e - s
        print(f"step {seq} {name:6s} ctas {len(v):4d}  start {s.min():8.1f} .. {np.median(s):8.1f} .. {s.max():8.1f}"
              f"  end {np.median(e):8.1f} .. {e.max():8.1f}  cta dur med {np.median(dur):6.1f} max {dur.max():6.1f}")
