"""Per-CTA timeline of a 20-step eca_pipeline_run (diagnostic build, ECA_TIMELINE):
where the first and last steps of a short stream lose time."""
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
eng.run_stream(pool, 0, 44)   # steps 0..43 (slots 0..43 mod 64 of the timeline buffer)
eng.fence()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
eng.run_stream(pool, 0, 20)   # steps 44..63
b.record(st)
torch.cuda.synchronize()
print(f"20 steps: {a.elapsed_time(b) * 1e3 / 20:.1f} us/step")
buf = (ctypes.c_ulonglong * (2 * 64 * 1024 * 2))()
fn = _lib.load().eca_debug_timeline
fn.argtypes = [ctypes.c_void_p]
assert fn(ctypes.cast(buf, ctypes.c_void_p)) == 0
t = np.array(buf, dtype=np.int64).reshape(2, 64, 1024, 2).astype(np.float64)
t0 = None
for seq in range(44, 64):
    for kind, name in ((0, "bounds"), (1, "fit")):
        v = t[kind, seq]
        v = v[(v[:, 0] > 0) & (v[:, 1] > 0)]
        if not len(v):
            continue
        if t0 is None:
            t0 = v[:, 0].min()
        s, e = (v[:, 0] - t0) / 1e3, (v[:, 1] - t0) / 1e3
        print(f"step {seq - 44:2d} {name:6s} ctas {len(v):4d} start {s.min():7.1f}..{s.max():7.1f}"
              f"  end {np.median(e):7.1f}..{e.max():7.1f}")
