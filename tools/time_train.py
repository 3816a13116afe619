"""EdgeNet training step time (bench train_leg workload: 2048 strips 5x7x1920,
batch 8): the public call's wall clock (bench.train_leg) and the device time
of one SGD step (forward + loss + backward + update), an epoch of 256 steps
captured as one CUDA graph and replayed, timed with CUDA events.

    python tools/time_train.py            # tcgen05 kernels
    ECA_TRAIN_SIMT=1 python tools/time_train.py
"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2210_14771_b200 as eb  # noqa: E402


if __name__ == "__main__":
    dev = torch.device("cuda", 0)
    tag = "simt" if os.environ.get("ECA_TRAIN_SIMT") == "1" else "tcgen05"
    x, t = bench._train_data(bench.TRAIN_M)
    us = bench.train_graph_step_us(eb, dev, torch.from_numpy(x).to(dev), torch.from_numpy(t).to(dev))
    print(f"{tag}: graph-replayed SGD step {us:.1f} us = {bench.TRAIN_BATCH / us * 1e6:.0f} samples/s")
    if "--api" in sys.argv:
        r = bench.train_leg(eb, dev)
        print(f"{tag}: edgenet.train {r['value']} samples/s ({r['ms_per_step'] * 1e3:.1f} us/step over 16 "
              f"epochs); device {r['device_us_per_step']} us/step")
