"""pseudo_label wall clock over 256 (or N) 1080p PNG frames of the C2 mix
with W decode workers.  usage: python tools/time_labels.py [N] [W ...]"""
import os
import sys
import tempfile
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_14771_b200 import labels  # noqa: E402

if __name__ == "__main__":   # (forkserver workers import this module)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ws = [int(a) for a in sys.argv[2:]] or [None]
    base = bench.base_frames(40)
    d = tempfile.mkdtemp(prefix="eca_tl_")
    for k in range(n):
        labels.save_image(base[k % len(base)], os.path.join(d, f"frame_{k:05d}.png"))
    for w in ws:
        labels.pseudo_label(d, chunk=64, workers=w)   # warm-up (pool start)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        anns = labels.pseudo_label(d, chunk=64, workers=w)
        dt = time.perf_counter() - t0
        print(f"workers {w or 'default'}: {len(anns) / dt:.1f} frames/s ({len(anns)} frames)")
