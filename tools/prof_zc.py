"""e2e from pinned host frames: strip-row H2D copies (run_host) vs zero-copy chunked reads."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
import bench
B = 256
base = bench.base_frames(40)
import numpy as np
host = torch.from_numpy(np.stack([base[i % 40] for i in range(B)])).pin_memory()
eng = eb.ContentAreaEngine(1080, 1920, B)
for fn, name in ((eng.run_host, "run_host (H2D strip rows)"), (eng.run_host_zero_copy, "zero-copy")):
    for _ in range(3): fn(host)
    b0 = eng.zero_copy_bytes()
    n = 20
    t0 = time.perf_counter()
    for _ in range(n): fn(host)
    dt = (time.perf_counter() - t0) / n
    mb = (eng.zero_copy_bytes() - b0) / n / 1e6
    print(f"{name:28s} {dt * 1e3:7.3f} ms/step  {B / dt:9.0f} frames/s  zero-copy MB/step {mb:.1f}")
# streamed: zero-copy reads + records D2H on the side stream, one sync at the end
recs = [torch.empty((B, 5), dtype=torch.float64).pin_memory() for _ in range(2)]
for i in range(4): eng.run_host_pipelined(host, recs[i % 2])
eng.fence(); torch.cuda.synchronize()
n = 20
t0 = time.perf_counter()
for i in range(n): eng.run_host_pipelined(host, recs[i % 2])
eng.fence(); torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / n
print(f"{'zero-copy pipelined':28s} {dt * 1e3:7.3f} ms/step  {B / dt:9.0f} frames/s")
ref = eng.run_host(host).clone()
assert torch.equal(recs[(n - 1) % 2], ref), "pipelined host records differ"
print("records match run_host")
