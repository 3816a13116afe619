"""Small ncu target: 3x engine.run (bounds + rescore + fit), or 3x engine.points with
argv[1] == "points", on a B=256 1080p batch."""
import sys, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
import bench
B = 256
dev = torch.device('cuda', 0)
base = bench.base_frames(40)
frames = torch.from_numpy(base[[i % 40 for i in range(B)]]).to(dev)
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
for _ in range(3):
    if sys.argv[1:] == ["points"]:
        eng.points(frames)
    else:
        eng.run(frames)
torch.cuda.synchronize()
print("ok")
