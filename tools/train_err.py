"""Error of the GPU training kernels vs the numpy FP32 oracle: logits and
per-layer gradients (max |diff| / max |want|), for the current path (tcgen05,
or SIMT with ECA_TRAIN_SIMT=1).

    python tools/train_err.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb  # noqa: E402
from oracle import eca_oracle as orc  # noqa: E402
from paper_2210_14771_b200 import training as tr  # noqa: E402

tag = "simt" if os.environ.get("ECA_TRAIN_SIMT") == "1" else "tc"
shapes = [(7, 40, 4), (7, 1920, 8), (11, 300, 2)]
if len(sys.argv) > 1:   # h,w,m triples: python tools/train_err.py 7,1920,64
    shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for (h, w, m) in shapes:
    rng = np.random.default_rng(h * w + m)
    x = rng.normal(0.0, 1.0, (m, 5, h, w)).astype(np.float32)
    t = rng.uniform(0.0, 1.0, (m, 1, h - 6, w - 6)).astype(np.float32)
    net = eb.EdgeNet(eb.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=4)
    layers = [(l.kernel, l.bias) for l in net.layers]
    wl, _ = orc.forward_logits(x, layers)
    gl = tr.forward_logits(net, x)
    loss, grads = tr.gradients(net, x, t)
    wloss, wgrads, _ = orc.train_step(x, t, layers, 0.0)
    errs = [np.abs(gl - wl).max() / np.abs(wl).max()]
    for (gk, gb), (wk, wb) in zip(grads, wgrads):
        errs += [np.abs(gk - wk).max() / np.abs(wk).max(), np.abs(gb - wb).max() / max(np.abs(wb).max(), 1e-30)]
    print(f"{tag} h={h} w={w} m={m}: loss rel {abs(loss - wloss) / wloss:.2e}; logits "
          + " ".join(f"{e:.1e}" for e in errs[:1]) + "; grads (w, b) per layer "
          + " ".join(f"{e:.1e}" for e in errs[1:]))
