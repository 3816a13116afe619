"""Golden fixtures for GPU pseudo-labelling, made by running the
REFERENCE's ``eca.dataset.pseudo_label`` (dataset.py:190-225) in the build
container on a directory of rendered frames:

    python tests/golden/make_golden_labels.py

Frames are not stored: labels.json keeps each frame's render recipe
(benchmark_specs(seed=2024) category + rng_seed, 320x240) and SHA-256; the GPU
test re-renders them with paper_2210_14771_b200.synth, writes the same PNG
directory (plus an unreadable file) and compares annotations.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from eca import dataset as ds  # noqa: E402

OUT = Path(__file__).resolve().parent
W, H, N = 320, 240, 9


def main():
    specs = ds.benchmark_specs(N, W, H, np.random.default_rng(2024))
    frames = [ds.render_synthetic(s, 40000 + k)[0] for k, (_, s) in enumerate(specs)]
    res = {"w": W, "h": H, "spec_seed": 2024, "rng_seed0": 40000,
           "sha256": [hashlib.sha256(f.tobytes()).hexdigest() for f in frames]}
    with tempfile.TemporaryDirectory() as d:
        for k, f in enumerate(frames):
            ds.save_image(f, Path(d) / f"frame_{k:04d}.png")
        (Path(d) / "frame_0004b.png").write_bytes(b"not an image")   # unreadable, skipped
        (Path(d) / "notes.txt").write_text("ignored")
        for name, kw in (("all", {}), ("fps1", {"fps": 1.0}), ("seed7", {"seed": 7, "video_no": 3,
                                                                         "source": ds.Source.CHOLEC80})):
            anns = ds.pseudo_label(d, **kw)
            res[name] = {"kw": {k: (v.value if hasattr(v, "value") else v) for k, v in kw.items()},
                         "anns": [[a.sample_id, a.source.value, a.video_no, a.frame_no,
                                   None if a.area is None else [a.area.cx, a.area.cy, a.area.r],
                                   a.image_path] for a in anns],
                         "csv": ds.dumps_annotations(anns)}
    (OUT / "labels.json").write_text(json.dumps(res))
    print({k: len(v["anns"]) for k, v in res.items() if isinstance(v, dict)})


if __name__ == "__main__":
    main()
