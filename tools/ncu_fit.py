"""ncu target: 3 x engine.run() (bounds + fit kernel with its rescore stage) on
a B=256 1080p C2 batch; profile with -k regex:fit_kernel."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb  # noqa: E402
from support import synth  # noqa: E402

B = 256
specs = synth.bench_specs(40, 1920, 1080, seed=2024)
base = np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])
frames = torch.from_numpy(base[[i % 40 for i in range(B)]]).cuda()
eng = eb.ContentAreaEngine(1080, 1920, B)
for _ in range(3):
    eng.run(frames)
torch.cuda.synchronize()
print("ok")
