"""EdgeNet training step time (bench train_leg workload: 2048 strips 5x7x1920,
batch 8): the public call's wall clock and the steady graph-replay step.

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
    r = bench.train_leg(eb, torch.device("cuda", 0))
    tag = "simt" if os.environ.get("ECA_TRAIN_SIMT") == "1" else "tcgen05"
    print(f"{tag}: {r['value']} samples/s ({r['ms_per_step'] * 1e3:.1f} us/step over 16 epochs); "
          f"steady {r['steady_us_per_step']} us/step = {r['steady_samples_per_s']} samples/s")
