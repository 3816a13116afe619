"""Bound-and-prune launch timing under the launch modes the engine uses:
back-to-back eca_bounds_handcrafted on alternating workspaces with flags
0 (plain), 1 (programmatic dependent launch), 2 (one CTA slot per SM left
free), 3 (both, as eca_pipeline_step), plus the pipelined step itself.
    python tools/prof_bounds.py [batch]"""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2210_14771_b200 as eb  # noqa: E402
from paper_2210_14771_b200 import _lib, api  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
NP = max(2048, 4 * B)
pool = torch.empty((NP, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(NP):
    pool[i].copy_(base[i % 40])
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
lib = _lib.load()
st = api._stream(dev)
S = eng.n_strips
ws = [torch.zeros_like(eng.workspace) for _ in range(2)]
outs = [(torch.empty_like(eng.xs), torch.empty_like(eng.ys), torch.empty_like(eng.sc)) for _ in range(2)]
nslot = NP // B


def bounds(i, flags):
    f = pool[(i % nslot) * B:][:B]
    o = outs[i & 1]
    _lib.check(lib.eca_bounds_handcrafted(api._ptr(f), B, f.stride(0), f.stride(1), eng._rows, None, S,
                                          ctypes.byref(eng.params), api._ptr(o[0]), api._ptr(o[1]),
                                          api._ptr(o[2]), api._ptr(ws[i & 1]), flags, st), "b")


def timeit(fn, n=200):
    for i in range(10):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


bytes_launch = B * 16 * 3 * 1920 * 3
import os
for fl in ((0,) if os.environ.get("QUICK") else (0, 1, 2, 3, 0, 1)):
    us = timeit(lambda i: bounds(i, fl))
    print(f"B={B} bounds only, flags={fl}: {us:6.1f} us/launch  {bytes_launch / us / 1e3:7.1f} GB/s")


def step(i):
    eng.run_pipelined(pool[(i % nslot) * B:][:B])


us = timeit(step)
eng.fence()
print(f"B={B} pipelined step: {us:6.1f} us  ({B / us:.2f} M frames/s)")

# the fitter alone on one batch's candidates (eca_fit)
eng.run(pool[:B])
trip = eng._trip if hasattr(eng, "_trip") else None
torch.cuda.synchronize()


def fit_only(i):
    _lib.check(lib.eca_fit(api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc), B, 2 * S,
                           ctypes.byref(eng.params), api._ptr(eng.trip), 0, api._ptr(eng.rec), st), "fit")


if hasattr(eng, "trip") and not os.environ.get("QUICK"):
    print(f"B={B} fit only: {timeit(fit_only):6.1f} us")
