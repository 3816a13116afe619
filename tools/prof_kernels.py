"""Time the pieces of the step separately on a B=256 1080p batch (rotating pool)."""
import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import _lib, api
import bench
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device('cuda', 0)
base = bench.base_frames(40)
pool = torch.empty((2048, 1080, 1920, 3), dtype=torch.uint8, device=dev)
bd = torch.from_numpy(base).to(dev)
for i in range(2048): pool[i].copy_(bd[i % 40])
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
lib = _lib.load(); st = api._stream(dev)
S = eng.n_strips
def frames(i): return pool[(i % (2048 // B)) * B:][:B]
def points(i, ws=True):
    f = frames(i)
    _lib.check(lib.eca_points_handcrafted(api._ptr(f), B, f.stride(0), f.stride(1), eng._rows, None, S, ctypes.byref(eng.params), api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc), api._ptr(eng.workspace) if ws else None, st), "pts")
def fit(i):
    _lib.check(lib.eca_fit(api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc), B, 2 * S, ctypes.byref(eng.params), api._ptr(eng.trip), 0, api._ptr(eng.rec), st), "fit")
def fused(i):
    f = frames(i)
    _lib.check(lib.eca_estimate_handcrafted(api._ptr(f), B, f.stride(0), f.stride(1), eng._rows, None, S, ctypes.byref(eng.params), api._ptr(eng.trip), api._ptr(eng.counters), api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc), api._ptr(eng.rec), st), "fused")
def timeit(fn, n=50):
    for i in range(5): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n): fn(i)
    eng.fence()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
for name, fn in [("points(2-stage)", points), ("points(1-kernel)", lambda i: points(i, False)), ("fit", fit), ("fused", fused), ("engine.run", lambda i: eng.run(frames(i))), ("run_pipelined", lambda i: eng.run_pipelined(frames(i)))]:
    ms = timeit(fn)
    print(f"{name:18s} B={B} {ms*1e3:9.1f} us  {ms*1e3/B:7.3f} us/frame  {70778880*B/256/(ms/1e3)/1e9:8.1f} GB/s(strip bytes)", flush=True)
