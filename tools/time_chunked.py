"""Device-resident frames through the bound-and-prune kernel's two staging
modes: whole half rows up front (default) vs scan chunks on demand
(ECA_BOUNDS_ZERO_COPY, reads only as far as the early exit lets the scan go)."""
import ctypes
import sys
import torch
sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2210_14771_b200 as eb  # noqa: E402
from paper_2210_14771_b200 import _lib, api  # noqa: E402

B = 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
pool = torch.empty((2048, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(2048):
    pool[i].copy_(base[i % 40])
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
lib = _lib.load()
wss = [torch.zeros_like(eng.workspace) for _ in range(4)]


def bounds(i, flags):
    f = pool[(i % 8) * B:][:B]
    _lib.check(lib.eca_bounds_handcrafted(api._ptr(f), B, f.stride(0), f.stride(1), eng._rows, None,
                                          eng.n_strips, ctypes.byref(eng.params), api._ptr(eng.xs),
                                          api._ptr(eng.ys), api._ptr(eng.sc), api._ptr(wss[i % 4]), flags,
                                          api._stream(dev)), "b")


a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fl in (("whole", 0), ("chunked", 4), ("whole+pdl", 1), ("chunked+pdl", 5)):
    for i in range(10):
        bounds(i, fl)
    torch.cuda.synchronize()
    a.record()
    for i in range(200):
        bounds(i, fl)
    b.record()
    torch.cuda.synchronize()
    print(f"{name:12s} {a.elapsed_time(b) / 200 * 1e3:6.2f} us")
