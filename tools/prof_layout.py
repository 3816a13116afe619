"""K1 timing: full-frame pool vs compact strip-row bands pool (same bytes read)."""
import sys, ctypes, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import _lib, api
import bench
B = 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
S = eng.n_strips
lib = _lib.load(); st = api._stream(dev)
NSLOT = 8
pool = torch.empty((NSLOT * B, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(NSLOT * B): pool[i].copy_(base[i % 40])
rows = eng.rows
bands = torch.empty((NSLOT * B, S * 3, 1920, 3), dtype=torch.uint8, device=dev)
for k, y in enumerate(rows):
    bands[:, 3 * k:3 * k + 3] = pool[:, y - 1:y + 2]
band_idx = api._i32_array([3 * k for k in range(S)])
def run_frames(i):
    f = pool[(i % NSLOT) * B:][:B]
    _lib.check(lib.eca_points_handcrafted(api._ptr(f), B, f.stride(0), f.stride(1), eng._rows, None, S, ctypes.byref(eng.params), api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc), api._ptr(eng.workspace), st), "f")
def run_bands(i):
    f = bands[(i % NSLOT) * B:][:B]
    _lib.check(lib.eca_points_handcrafted(api._ptr(f), B, f.stride(0), f.stride(1), eng._rows, band_idx, S, ctypes.byref(eng.params), api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc), api._ptr(eng.workspace), st), "b")
def timeit(fn, n=50):
    for i in range(5): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n): fn(i)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
tf = timeit(run_frames); xf = eng.xs.clone()
tb = timeit(run_bands); xb = eng.xs.clone()
print(f"frames pool {tf:.1f} us   bands pool {tb:.1f} us   same candidates: {torch.equal(xf, xb)}")
