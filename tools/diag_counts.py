"""Histogram of bounds_kernel survivor counts per half row (-1 = resolved in-kernel)."""
import sys, collections, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
import bench
B = 256
dev = torch.device('cuda', 0)
base = bench.base_frames(40)
frames = torch.from_numpy(base[[i % 40 for i in range(B)]]).to(dev)
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
eng.points(frames)
torch.cuda.synchronize()
n_hr = B * eng.n_strips * 2
slots = n_hr * 8 * 24
off = (slots + 255) & ~255
counts = eng.workspace[off:off + 4 * n_hr].view(torch.int32).cpu().tolist()
h = collections.Counter(counts)
print(sorted(h.items()))
neg = [i for i, c in enumerate(counts) if c < 0]
print("resolved in-kernel:", len(neg), "first:", [(i // 2 // eng.n_strips % 40, i // 2 % eng.n_strips, i & 1) for i in neg[:20]])
