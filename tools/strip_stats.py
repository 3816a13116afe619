"""Diagnostic: survivor / pruning / stall statistics of the strip kernel on the C2 batch.
Needs the ECA_STATS build (tools/build_stats.sh -> build/libeca_stats.so)."""
import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import api
import bench
lib = ctypes.CDLL("build/libeca_stats.so")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device('cuda', 0)
base = bench.base_frames(40)
frames = torch.from_numpy(base[[i % 40 for i in range(B)]]).to(dev)
rows = eb.strip_heights(1080, 16, 8.0)
p = eb.EcaConfig().device_params(1920, 1080)
xs = torch.empty((B, 32), dtype=torch.int32, device=dev); ys = torch.empty_like(xs); sc = torch.empty((B, 32), dtype=torch.float64, device=dev)
out = (ctypes.c_ulonglong * 16)()
def run():
    return lib.eca_points_handcrafted(ctypes.c_void_p(frames.data_ptr()), B, ctypes.c_int64(frames.stride(0)), ctypes.c_int64(frames.stride(1)), api._i32_array(rows), None, 16, ctypes.byref(p), ctypes.c_void_p(xs.data_ptr()), ctypes.c_void_p(ys.data_ptr()), ctypes.c_void_p(sc.data_ptr()), None)
run(); torch.cuda.synchronize()
lib.eca_debug_strip_stats(out, 1)
rc = run(); torch.cuda.synchronize()
lib.eca_debug_strip_stats(out, 0)
o = list(out); items = o[0]
print(f"rc={rc} items={items} survivors/item={o[1]/items:.2f} max={o[5]} looking/item={o[2]/items:.2f} of {o[3]/items:.1f} full/item={o[4]/items:.3f}")
print(f"cycles per item: pixel TMA wait {o[6]/items:.0f}, pixel wait free {o[7]/items:.0f}, pixel item {o[8]/items:.0f}, fp64 wait ready {o[9]/items:.0f}, fp64 item {o[10]/items:.0f}")
