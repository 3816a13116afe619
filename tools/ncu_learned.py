"""ncu target: one learned step (B=64) with the tensor-core CNN variant."""
import sys, torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
import bench
B = 64
dev = torch.device('cuda', 0)
frames = torch.from_numpy(bench.base_frames(40)[[i % 40 for i in range(B)]]).to(dev)
net = eb.EdgeNet(eb.ChannelStats([100.0] * 3, [50.0] * 3), seed=0)
for tc in (True, False):
    eng = eb.ContentAreaEngine(1080, 1920, B, variant=eb.Learned(net), device=dev, tensor_cores=tc)
    eng.run(frames)
torch.cuda.synchronize()
print("ok")
