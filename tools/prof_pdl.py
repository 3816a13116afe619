"""Back-to-back eca_bounds_handcrafted launches on alternating workspaces,
without and with ECA_BOUNDS_OVERLAP_PREVIOUS (programmatic dependent launch)."""
import sys, ctypes, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import _lib, api
import bench
B = 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
pool = torch.empty((2048, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(2048): pool[i].copy_(base[i % 40])
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
lib = _lib.load(); st = api._stream(dev)
S = eng.n_strips
ws = [torch.zeros_like(eng.workspace) for _ in range(2)]
outs = [(torch.empty_like(eng.xs), torch.empty_like(eng.ys), torch.empty_like(eng.sc)) for _ in range(2)]
def bounds(i, flags):
    f = pool[(i % 8) * B:][:B]
    o = outs[i & 1]
    _lib.check(lib.eca_bounds_handcrafted(api._ptr(f), B, f.stride(0), f.stride(1), eng._rows, None, S, ctypes.byref(eng.params), api._ptr(o[0]), api._ptr(o[1]), api._ptr(o[2]), api._ptr(ws[i & 1]), flags, st), "b")
def timeit(fn, n=100):
    for i in range(6): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n): fn(i)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
for fl in (0, 2, 0, 2):
    print(f"bounds only, flags={fl}: {timeit(lambda i: bounds(i, fl)):.1f} us/launch")
