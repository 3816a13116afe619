"""Per-warp timeline of one bounds_kernel launch.  Needs a diagnostic build:
    ECA_NVCC_DEFINES=-DECA_WARP_TIMES python -m paper_2210_14771_b200.build --force
"""
import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import _lib
import bench
B = 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
pool = torch.empty((512, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(512): pool[i].copy_(base[i % 40])
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
for i in range(3): eng.points(pool[(i % 2) * B:][:B])
torch.cuda.synchronize()
n = 740 * 4
buf = (ctypes.c_uint64 * (3 * n))()
lib = _lib.load()
lib.eca_debug_warp_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.eca_debug_warp_times(buf, n) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 3).astype(np.float64)
t0 = a[:, 0].min()
st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
print(f"warps {n}: start max {st.max():.1f} us; end min {en.min():.1f} / p10 {np.percentile(en,10):.1f} / "
      f"p50 {np.median(en):.1f} / p90 {np.percentile(en,90):.1f} / max {en.max():.1f} us")
# slowest item per warp: duration, full flag, step-C groups, item -> (frame, strip, half)
rec = np.frombuffer(buf, dtype=np.uint64).reshape(n, 3)[:, 2]
dur = (rec >> np.uint64(40)).astype(np.float64) * 32 / 1e3
full = (rec >> np.uint64(39)) & np.uint64(1)
grp = (rec >> np.uint64(32)) & np.uint64(127)
item = (rec & np.uint64(0xffffffff)).astype(np.int64)
order = np.argsort(-dur)[:25]
S = eng.n_strips
for k in order:
    it = int(item[k]); fr = it // 2 // S
    print(f"{dur[k]:6.1f} us  full {int(full[k])}  groups {int(grp[k]):3d}  frame {fr} (cat {fr % 40 % 5})  strip {it // 2 % S}  half {it & 1}")
print("item duration percentiles (slowest per warp):", np.percentile(dur, [10, 50, 90, 99]).round(1))
