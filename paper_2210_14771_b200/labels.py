"""GPU pseudo-labelling: the paper's PseudoECA generator.

Drop-in for ``eca.dataset.pseudo_label`` (dataset.py:190-225) and the
annotation record it returns (dataset.py:36-60; its CSV file form, :63-81,
is host-side dataset tooling and out of scope).  The
reference decodes and estimates one frame at a time; here worker processes
decode the images and hand back only the strip rows the scorer reads, while
the GPU estimates the previous chunk, and each chunk of same-sized frames is
ONE batched launch sequence over those rows, so a directory of frames is
labelled at the decoder's speed.  Results are the reference's: the same handcrafted estimate
with the same seed per frame, the same frame numbering, stride and skipping.
"""

from __future__ import annotations

import logging
import os
import multiprocessing as mp
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass
from enum import Enum
from pathlib import Path

import numpy as np
import torch
from PIL import Image

from .api import (_device, _DevFrames, _handcrafted_batch, _i32_array, _ptr, _records_to_results,
                  strip_heights, validate_frame)
from .params import EcaConfig, config_default
from .shapes import Circle, CircularArea

LOGGER = logging.getLogger("paper_2210_14771_b200.labels")
IMAGE_EXTENSIONS = {".png", ".jpg", ".jpeg", ".bmp"}   # dataset.py:29


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
    """uint8 RGB (H, W, 3), as dataset.load_image (an RGB image is not
    converted: one copy out of the decoder instead of two)."""
    with Image.open(path) as im:
        return np.asarray(im if im.mode == "RGB" else im.convert("RGB"))


def save_image(frame: np.ndarray, path) -> None:
    Image.fromarray(frame, mode="RGB").save(path)


def _decode_bands(args):
    """Worker process: decode one image and keep only the rows the
    handcrafted scorer reads (y-1..y+1 of every strip row, handcrafted.py:
    167-169): ~0.3 MB instead of 6 MB per 1080p frame crosses back."""
    path, count, weighting = args
    try:
        frame = load_image(path)
    except OSError as exc:
        return None, None, exc
    h, w = frame.shape[:2]
    try:   # malformed frame: the reference's estimate() raises (strips.py:13-27)
        validate_frame(frame)
        rows = strip_heights(h, count, weighting)
    except ValueError as exc:
        return (h, w), None, exc
    idx = np.concatenate([[r - 1, r, r + 1] for r in rows])
    return (h, w), np.ascontiguousarray(frame[idx]), None


def _estimate_bands(bands: np.ndarray, h: int, w: int, cfg: EcaConfig, seed: int, dev):
    """Fit records of a (B, 3S, W, 3) stack of strip-row bands (band k holds
    rows y_k-1..y_k+1): the eca_h2d_bands layout the kernels read directly."""
    rows = strip_heights(h, cfg.strip_count, cfg.strip_weighting)
    t = torch.from_numpy(bands).pin_memory().to(dev, non_blocking=True)
    band = _i32_array([3 * k for k in range(len(rows))])
    df = _DevFrames(_ptr(t), t.shape[0], t.stride(0), t.stride(1), band, t)
    return _handcrafted_batch(df, w, h, rows, cfg, seed, dev)[3]


_POOL: dict = {}


def _decode_pool(workers: int) -> ProcessPoolExecutor:
    """The decode workers, started once per process and reused by later calls.
    Forkserver, not fork: this process has CUDA and torch threads running, and
    a fork would copy their locks; the server is a clean single-threaded
    process that imports this module once, so workers start fast and never
    initialise CUDA (they only decode and compute strip rows)."""
    pool = _POOL.get(workers)
    if pool is None:
        ctx = mp.get_context("forkserver")
        ctx.set_forkserver_preload([__name__])
        pool = ProcessPoolExecutor(workers, mp_context=ctx)
        _POOL[workers] = pool
    return pool


def pseudo_label(frames_dir, cfg: EcaConfig | None = None, seed: int = 0,
                 source: Source = Source.SYNTHETIC, video_no: int = 0, fps: float | None = None,
                 *, chunk: int = 256, workers: int | None = None, device=None) -> list[EcaAnnotation]:
    """Label every readable frame in a directory with the handcrafted estimator
    (dataset.py:190-225).  Plain directories are labelled exhaustively; with
    ``fps`` the sorted files are consecutive video frames sampled once every
    two seconds.  Unreadable files are skipped with a log entry.

    Worker processes decode the frames and return only their strip rows;
    every ``chunk`` decoded frames (grouped by size) are one batched GPU
    estimate while the workers keep decoding."""
    cfg = cfg or config_default()
    frames_dir = Path(frames_dir)
    paths = sorted(p for p in frames_dir.iterdir() if p.suffix.lower() in IMAGE_EXTENSIONS)
    stride = max(1, round(2.0 * fps)) if fps else 1
    todo = [(n, p) for n, p in enumerate(paths) if n % stride == 0]
    out: list[EcaAnnotation] = []
    skipped = 0
    # every core decodes: this process only unpickles rows and launches the
    # GPU estimates (measured: 16 workers 355 vs 15 workers 336 frames/s on 16 cores)
    workers = workers or max(1, min(32, os.cpu_count() or 1))
    dev = _device(device)

    def label(batch, decoded):
        nonlocal skipped
        groups: dict = {}
        for (n, p), (shape, bands, err) in zip(batch, decoded):
            if bands is None:
                if isinstance(err, OSError):
                    LOGGER.warning("skipping unreadable frame %s: %s", p, err)
                    skipped += 1
                    continue
                raise err
            groups.setdefault(shape, []).append((n, p, bands))
        results = {}
        for (h, w), items in groups.items():
            rec = _estimate_bands(np.stack([b for _, _, b in items]), h, w, cfg, seed, dev)
            for (n, p, _), area in zip(items, _records_to_results(rec)):
                results[n] = (p, area)
        for n in sorted(results):
            p, area = results[n]
            circle = area.circle if isinstance(area, CircularArea) else None
            out.append(EcaAnnotation(p.stem, source, video_no, n, circle, p.name))

    # processes, not threads: PIL's decode and RGB conversion hold the GIL for
    # part of every frame; the workers never touch CUDA
    # every file is queued at once so no worker idles at chunk boundaries;
    # results arrive in order and are estimated chunk by chunk as they come
    # (the GPU is far faster than the decoders, so few results wait)
    results = _decode_pool(workers).map(
        _decode_bands, [(p, cfg.strip_count, cfg.strip_weighting) for _, p in todo], chunksize=2)
    batch, decoded = [], []
    for item, res in zip(todo, results):
        batch.append(item)
        decoded.append(res)
        if len(batch) == chunk:
            label(batch, decoded)
            batch, decoded = [], []
    if batch:
        label(batch, decoded)
    if skipped:
        LOGGER.warning("pseudo-labelling skipped %d unreadable frames", skipped)
    return out
