"""Host enqueue cost of one run_pipelined() step vs its GPU time (B=256 1080p)."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
import bench
B = 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
pool = torch.empty((2048, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(2048): pool[i].copy_(base[i % 40])
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
def fr(i): return pool[(i % 8) * B:][:B]
for i in range(20): eng.run_pipelined(fr(i))
eng.fence(); torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for i in range(n): eng.run_pipelined(fr(i))
t1 = time.perf_counter()
eng.fence(); torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {(t1 - t0) / n * 1e6:.1f} us/step; wall incl. drain {(t2 - t0) / n * 1e6:.1f} us/step")
# the native call alone, arguments prepared once
import ctypes
from paper_2210_14771_b200 import _lib
p = eng._pipeline()
lib = _lib.load()
args = [(ctypes.c_void_p(fr(i).data_ptr()), fr(i).stride(0), fr(i).stride(1)) for i in range(8)]
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
out = ctypes.c_void_p()
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    a = args[i % 8]
    lib.eca_pipeline_step(p["handle"], a[0], a[1], a[2], st, ctypes.byref(out))
t1 = time.perf_counter()
eng.fence(); torch.cuda.synchronize()
print(f"native eca_pipeline_step alone: {(t1 - t0) / n * 1e6:.1f} us/step")
t0 = time.perf_counter()
for i in range(n):
    torch.cuda.current_stream(dev)
t1 = time.perf_counter()
print(f"torch.cuda.current_stream: {(t1 - t0) / n * 1e6:.2f} us; ", end="")
f = fr(0)
t0 = time.perf_counter()
for i in range(n):
    eng._check_frames(f)
t1 = time.perf_counter()
print(f"_check_frames: {(t1 - t0) / n * 1e6:.2f} us")
