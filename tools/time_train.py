"""EdgeNet training step time (bench train_leg workload): 4 epochs of 2048
strips 5x7x1920, batch 8; run once with the tcgen05 kernels and once with
ECA_TRAIN_SIMT=1 (separate processes: the switch is read once).

    python tools/time_train.py [simt]
"""
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2210_14771_b200 as eb  # noqa: E402

if __name__ == "__main__":
    dev = torch.device("cuda", 0)
    r = bench.train_leg(eb, dev)
    tag = "simt" if os.environ.get("ECA_TRAIN_SIMT") == "1" else "tcgen05"
    print(f"{tag}: {r['value']} samples/s, {r['ms_per_step'] * 1e3:.1f} us/step")
