"""GPU pseudo-labelling: the paper's PseudoECA generator.

Drop-in for ``eca.dataset.pseudo_label`` (dataset.py:190-225) and the
annotation record it returns (dataset.py:36-60, CSV form :63-81).  The
reference decodes and estimates one frame at a time; here host threads decode
the images (PIL releases the GIL while decoding) while the GPU estimates the
previous chunk, and each chunk of same-sized frames is ONE batched launch
sequence (``estimate_batch``), so a directory of frames is labelled at the
decoder's speed.  Results are the reference's: the same handcrafted estimate
with the same seed per frame, the same frame numbering, stride and skipping.
"""

from __future__ import annotations

import csv
import io
import logging
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from enum import Enum
from pathlib import Path

import numpy as np
from PIL import Image

from .api import HANDCRAFTED, FrameError, estimate_batch
from .params import EcaConfig, config_default
from .shapes import Circle, CircularArea

LOGGER = logging.getLogger("paper_2210_14771_b200.labels")
IMAGE_EXTENSIONS = {".png", ".jpg", ".jpeg", ".bmp"}   # dataset.py:29
CSV_FIELDS = ("sample_id", "source", "video_no", "frame_no", "area_type", "cx", "cy", "r",
              "image_path")


class Source(Enum):   # dataset.py:44-47
    CHOLEC80 = "Cholec80"
    ROBUST_MIS = "RobustMIS"
    SYNTHETIC = "Synthetic"


@dataclass(frozen=True, slots=True)
class EcaAnnotation:
    """One annotated sample; ``area`` None means the full frame is content."""
    sample_id: str
    source: Source
    video_no: int
    frame_no: int
    area: Circle | None
    image_path: str


def load_image(path) -> np.ndarray:
    """uint8 RGB (H, W, 3), as dataset.load_image."""
    with Image.open(path) as im:
        return np.asarray(im.convert("RGB"))


def save_image(frame: np.ndarray, path) -> None:
    Image.fromarray(frame, mode="RGB").save(path)


def dumps_annotations(annotations) -> str:
    """The reference's flat CSV (dataset.py:63-77)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_FIELDS)
    for a in annotations:
        geo = ("full", "", "", "") if a.area is None else \
            ("circle", repr(a.area.cx), repr(a.area.cy), repr(a.area.r))
        w.writerow((a.sample_id, a.source.value, a.video_no, a.frame_no, *geo, a.image_path))
    return buf.getvalue()


def save_annotations(annotations, path) -> None:
    Path(path).write_text(dumps_annotations(annotations), encoding="utf-8")


def _decode(path):
    try:
        return load_image(path), None
    except OSError as exc:
        return None, exc


def pseudo_label(frames_dir, cfg: EcaConfig | None = None, seed: int = 0,
                 source: Source = Source.SYNTHETIC, video_no: int = 0, fps: float | None = None,
                 *, chunk: int = 256, workers: int | None = None, device=None) -> list[EcaAnnotation]:
    """Label every readable frame in a directory with the handcrafted estimator
    (dataset.py:190-225).  Plain directories are labelled exhaustively; with
    ``fps`` the sorted files are consecutive video frames sampled once every
    two seconds.  Unreadable files are skipped with a log entry.

    ``chunk`` frames are decoded ahead (``workers`` threads) and estimated as
    one GPU batch while the next chunk decodes."""
    cfg = cfg or config_default()
    frames_dir = Path(frames_dir)
    paths = sorted(p for p in frames_dir.iterdir() if p.suffix.lower() in IMAGE_EXTENSIONS)
    stride = max(1, round(2.0 * fps)) if fps else 1
    todo = [(n, p) for n, p in enumerate(paths) if n % stride == 0]
    out: list[EcaAnnotation] = []
    skipped = 0
    workers = workers or min(32, os.cpu_count() or 1)

    def label(batch, decoded):
        nonlocal skipped
        frames, keep = [], []
        for (n, p), (img, err) in zip(batch, decoded):
            if err is not None:
                LOGGER.warning("skipping unreadable frame %s: %s", p, err)
                skipped += 1
                continue
            frames.append(img)
            keep.append((n, p))
        if not frames:
            return
        areas = estimate_batch(frames, HANDCRAFTED, cfg, seed, device=device)
        for (n, p), a in zip(keep, areas):
            if isinstance(a, FrameError):
                raise ValueError(a.message)   # the reference's estimate() raises here
            circle = a.circle if isinstance(a, CircularArea) else None
            out.append(EcaAnnotation(p.stem, source, video_no, n, circle, p.name))

    with ThreadPoolExecutor(workers) as pool:
        chunks = [todo[i:i + chunk] for i in range(0, len(todo), chunk)]
        pending = pool.map(_decode, [p for _, p in chunks[0]]) if chunks else None
        for k, batch in enumerate(chunks):
            decoded = list(pending)
            if k + 1 < len(chunks):   # decode the next chunk while this one estimates
                pending = pool.map(_decode, [p for _, p in chunks[k + 1]])
            label(batch, decoded)
    if skipped:
        LOGGER.warning("pseudo-labelling skipped %d unreadable frames", skipped)
    return out
