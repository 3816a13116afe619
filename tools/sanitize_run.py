"""Small workload exercising every handcrafted / learned / mask / crop device
path once, for compute-sanitizer (tools/sanitize.sh): the pipelined stream
(bounds + fit with programmatic dependent launches and the device-side set
guard, zero-copy host reads), the latency path (in-warp rescore + fit), the
block-per-strip kernels (fused fit and score rows: named barriers), the
split bounds + rescore stages, the tcgen05 and SIMT CNNs, masks and crops."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb  # noqa: E402
from support import synth  # noqa: E402

W, H = 640, 480
specs = synth.bench_specs(40, W, H, seed=2024)
frames = np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])
dev = torch.from_numpy(frames).cuda()
B = 20
# pipelined stream over a 2-batch pool (4 buffer sets: set reuse exercised)
eng = eb.ContentAreaEngine(H, W, B)
pool = dev[:2 * B].contiguous()
eng.run_stream(pool, 0, 6)
for i in range(3):
    eng.run_pipelined(pool[(i % 2) * B:(i % 2 + 1) * B])            # griddepcontrol.wait path
eng.fence()
want = eng.run(pool[:B]).clone()
host = torch.from_numpy(frames[:B]).pin_memory()
rec = torch.zeros((B, 5), dtype=torch.float64).pin_memory()
eng.run_host_pipelined(host, rec)                                  # zero-copy TMA from pinned memory
eng.fence()
torch.cuda.synchronize()
assert torch.equal(rec, want.cpu())
eng.points(pool[:B])                                                # bounds + rescore kernels
# latency path (bounds in-warp rescore + fit) and the block-per-strip kernels
a = eb.estimate(frames[0])
os.environ["ECA_LATENCY_STRIP"] = "1"
b = eb.estimate_batch([frames[0]])[0]
del os.environ["ECA_LATENCY_STRIP"]
assert a == b, (a, b)
rows, _ = eb.score_frame_strips(frames[1])
# learned variant: tcgen05 and SIMT CNNs
net = eb.EdgeNet(eb.ChannelStats([100.0] * 3, [50.0] * 3), seed=0)
le = eb.ContentAreaEngine(H, W, 4, variant=eb.Learned(net))
r1 = le.run(dev[:4]).clone()
ls = eb.ContentAreaEngine(H, W, 4, variant=eb.Learned(net), tensor_cores=False)
r2 = ls.run(dev[:4]).clone()
# mask + crop
areas = eng.results(want)
m = eb.draw_mask(areas[:4], H, W)
c = eb.crop_area(dev[0], areas[0])
torch.cuda.synchronize()
print("sanitize workload ok:", a, m.shape, None if c is None else tuple(c.shape))
