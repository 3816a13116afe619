"""us per bound-and-prune launch, back to back with programmatic dependent
launch on 4 rotating workspaces (the pipeline's launch mode), B=256 1080p."""
import sys
import torch
sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2210_14771_b200 as eb  # noqa: E402

B = 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
pool = torch.empty((2048, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(2048):
    pool[i].copy_(base[i % 40])
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for overlap in (True, False):
    for i in range(20):
        eng.bounds(pool[(i % 8) * B:][:B], overlap=overlap, slot=i % 4)
    torch.cuda.synchronize()
    a.record()
    for i in range(300):
        eng.bounds(pool[(i % 8) * B:][:B], overlap=overlap, slot=i % 4)
    b.record()
    torch.cuda.synchronize()
    res.append(a.elapsed_time(b) / 300 * 1e3)
print(f"pdl {res[0]:6.2f} us  isolated {res[1]:6.2f} us")
