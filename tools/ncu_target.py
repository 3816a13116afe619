"""Small ncu target: 3x points-only, 3x fused estimate on a B=256 1080p batch."""
import sys, ctypes, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import _lib, api
import bench
B = 256
dev = torch.device('cuda', 0)
base = bench.base_frames(40)
frames = torch.from_numpy(base[[i % 40 for i in range(B)]]).to(dev)
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
lib = _lib.load(); st = api._stream(dev)
which = sys.argv[1] if len(sys.argv) > 1 else "both"
for _ in range(3):
    if which in ("points", "both"):
        _lib.check(lib.eca_points_handcrafted(api._ptr(frames), B, frames.stride(0), frames.stride(1), eng._rows, None, eng.n_strips, ctypes.byref(eng.params), api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc), st), "pts")
    if which in ("fused", "both"):
        eng.run(frames)
torch.cuda.synchronize()
print("ok")
