"""Learned variant (C3): EdgeNet strip CNN + selection + fit on 256 x 1080p frames."""
import sys, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
import bench
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
pool = torch.empty((2 * B, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(2 * B): pool[i].copy_(base[i % 40])
net = eb.EdgeNet(eb.ChannelStats([100.0] * 3, [50.0] * 3), seed=0)
eng = eb.ContentAreaEngine(1080, 1920, B, variant=eb.Learned(net), device=dev)
def timeit(fn, n=10):
    for i in range(2): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n): fn(i)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
ms = timeit(lambda i: eng.run(pool[(i % 2) * B:][:B]))
flop = 606.6e6 * B
print(f"learned estimate B={B}, default (tcgen05 CNN): {ms * 1e3:.1f} us/step  {B / ms * 1e3:.0f} frames/s  "
      f"CNN {flop / (ms * 1e-3) / 1e12:.1f} TFLOP/s")
eng_simt = eb.ContentAreaEngine(1080, 1920, B, variant=eb.Learned(net), device=dev, tensor_cores=False)
ms = timeit(lambda i: eng_simt.run(pool[(i % 2) * B:][:B]))
print(f"learned estimate B={B}, SIMT CNN: {ms * 1e3:.1f} us/step  {B / ms * 1e3:.0f} frames/s  "
      f"CNN {flop / (ms * 1e-3) / 1e12:.1f} TFLOP/s")
