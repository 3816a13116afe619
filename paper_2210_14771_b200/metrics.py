"""Normalised-Hausdorff evaluation of content areas on the GPU.

Drop-in for ``eca.metrics`` (metrics.py:1-283).  Boundary sampling and the
Hausdorff distance run in libeca_b200.so (csrc/eca_eval.cu): the boundary of
disk ∩ frame is sampled on the device exactly as ``boundary_points`` does, and
the directed distances are exact FP64 nearest-neighbour maxima (the reference
uses a KD-tree; the minimum / maximum are the same numbers).  Aggregation
(mean, miss percentages, the markdown table) stays on the host like the
reference's.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from enum import Enum
from typing import Mapping

import numpy as np
import torch

from . import _lib
from .api import _area_records, _device, _ptr, _stream
from .shapes import Circle, CircularArea, ContentArea, FullFrame

REF_DIAGONAL = math.hypot(1920.0, 1080.0)   # metrics.py:23
HIT_MAX_NH_PX = 15.0
MISS_MAX_NH_PX = 25.0


class MissClass(Enum):
    HIT = "hit"
    MISS = "miss"
    BAD_MISS = "bad_miss"


def classify(nh: float) -> MissClass:
    """metrics.py:34-39: above 25 px a bad miss, above 15 px a miss."""
    if nh > MISS_MAX_NH_PX:
        return MissClass.BAD_MISS
    return MissClass.MISS if nh > HIT_MAX_NH_PX else MissClass.HIT


def as_circle(area) -> Circle | None:
    """metrics.py:42-50: None means full frame."""
    if area is None or isinstance(area, FullFrame):
        return None
    if isinstance(area, CircularArea):
        return area.circle
    if isinstance(area, Circle):
        return area
    raise TypeError(f"not a content area: {area!r}")


def _check_dims(width: int, height: int) -> None:
    if width < 2 or height < 2:
        raise ValueError(f"degenerate frame {width}x{height}")


def _boundary_cap(width: int, height: int, spacing: float) -> int:
    # eca_eval.cu boundary_cap: perimeter / spacing + 2 per piece + slack
    return int(math.ceil(2.0 * ((width - 1) + (height - 1)) / spacing)) + 2 * 12 + 64


def boundary_points(area, width: int, height: int, spacing: float = 1.0, device=None) -> np.ndarray:
    """metrics.py:148-176 on the GPU: (n, 2) float64 points along the border of
    disk ∩ [0, W-1] x [0, H-1], arcs first, then the covered edge runs."""
    _check_dims(width, height)
    circle = as_circle(area)
    if not spacing > 0.0:
        raise ValueError(f"spacing must be positive, got {spacing}")
    dev = _device(device)
    rec = _area_records([circle], dev)
    cap = _boundary_cap(width, height, spacing)
    out = torch.empty((cap, 2), dtype=torch.float64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().eca_boundary_points(_ptr(rec), width, height, float(spacing), _ptr(out),
                                               cap, _ptr(cnt), _stream(dev)), "eca_boundary_points")
    n = int(cnt.item())
    if n == 0:
        raise ValueError(f"{circle} does not intersect a {width}x{height} frame")
    if n > cap:
        raise _lib.EcaError(f"eca_boundary_points: {n} samples exceed the bound {cap}")
    return out[:n].cpu().numpy()


def _arcs(circle: Circle, width: int, height: int) -> list[tuple[float, float]]:
    """Angular intervals of the circle inside the frame (metrics.py:52-88)."""
    cx, cy, r = circle.cx, circle.cy, circle.r
    xhi, yhi = float(width - 1), float(height - 1)
    two_pi = 2.0 * math.pi
    cross = []
    for b in (0.0, xhi):
        c = (b - cx) / r
        if -1.0 <= c <= 1.0:
            t = math.acos(c)
            cross += [t, two_pi - t]
    for b in (0.0, yhi):
        s = (b - cy) / r
        if -1.0 <= s <= 1.0:
            t = math.asin(s)
            cross += [t % two_pi, (math.pi - t) % two_pi]

    def inside(t):
        x, y = cx + r * math.cos(t), cy + r * math.sin(t)
        return 0.0 <= x <= xhi and 0.0 <= y <= yhi

    if not cross:
        return [(0.0, two_pi)] if inside(0.0) else []
    ts = sorted(set(cross))
    out = []
    for k, t0 in enumerate(ts):
        t1 = ts[k + 1] if k + 1 < len(ts) else ts[0] + two_pi
        if t1 - t0 > 1e-12 and inside((t0 + t1) / 2.0):
            out.append((t0, t1))
    return out


def _edge_runs(circle: Circle, width: int, height: int) -> list[float]:
    """Lengths of the frame-edge runs covered by the disk (metrics.py:91-118)."""
    cx, cy, r = circle.cx, circle.cy, circle.r
    xhi, yhi = float(width - 1), float(height - 1)
    out = []
    for fixed, hi, horizontal in ((0.0, xhi, True), (yhi, xhi, True), (0.0, yhi, False),
                                  (xhi, yhi, False)):
        rad2 = r * r - ((fixed - cy) ** 2 if horizontal else (fixed - cx) ** 2)
        if rad2 < 0.0:
            continue
        half = math.sqrt(rad2)
        mid = cx if horizontal else cy
        a, b = max(0.0, mid - half), min(hi, mid + half)
        if b > a:
            out.append(b - a)
    return out


def boundary_length(area, width: int, height: int) -> float:
    """Analytic boundary length (metrics.py:179-190); host scalar geometry."""
    circle = as_circle(area)
    if circle is None:
        return 2.0 * float(width - 1 + height - 1)
    arcs = sum(circle.r * (t1 - t0) for t0, t1 in _arcs(circle, width, height))
    return arcs + sum(_edge_runs(circle, width, height))


def _as_points(a) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a, dtype=np.float64))
    t = t.to(torch.float64)
    if t.ndim != 2 or t.shape[1] != 2:
        t = t.reshape(-1, 2)
    return t


def hausdorff(a, b, device=None) -> float:
    """Symmetric Hausdorff distance of two 2-D point sets (metrics.py:193-203),
    exact FP64 on the GPU."""
    ta, tb = _as_points(a), _as_points(b)
    if len(ta) == 0 or len(tb) == 0:
        raise ValueError("hausdorff distance needs non-empty point sets")
    dev = _device(device)
    ta, tb = ta.to(dev).contiguous(), tb.to(dev).contiguous()
    lib = _lib.load()
    nbytes = ctypes.c_int64()
    _lib.check(lib.eca_hausdorff_workspace_bytes(max(len(ta), len(tb)), ctypes.byref(nbytes)),
               "eca_hausdorff_workspace_bytes")
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    hd = torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.check(lib.eca_hausdorff_points(_ptr(ta), len(ta), _ptr(tb), len(tb), _ptr(ws), nbytes.value,
                                        _ptr(hd), _ptr(st), _stream(dev)), "eca_hausdorff_points")
    return float(hd.item())


def normalized_hausdorff(a, b, width: int, height: int, device=None) -> float:
    """Hausdorff distance scaled to a 1920x1080 reference diagonal (metrics.py:206-208)."""
    return REF_DIAGONAL / math.hypot(width, height) * hausdorff(a, b, device)


def area_errors(predictions, truths, frame_dims, spacing: float = 1.0, device=None) -> np.ndarray:
    """Batched ``area_error_px``: NH of every (prediction, truth) pair in one
    set of launches.  ``frame_dims`` is one (width, height) or one per pair."""
    preds, truths = list(predictions), list(truths)
    if len(preds) != len(truths):
        raise ValueError(f"{len(preds)} predictions for {len(truths)} truths")
    n = len(preds)
    if n == 0:
        return np.zeros(0)
    dims = np.asarray(frame_dims, dtype=np.int64).reshape(-1, 2)
    if len(dims) == 1:
        dims = np.repeat(dims, n, axis=0)
    if len(dims) != n:
        raise ValueError(f"{len(dims)} frame sizes for {n} samples")
    for w, h in dims:
        _check_dims(int(w), int(h))
    if not spacing > 0.0:
        raise ValueError(f"spacing must be positive, got {spacing}")
    dev = _device(device)
    rp = _area_records([as_circle(a) for a in preds], dev)
    rt = _area_records([as_circle(a) for a in truths], dev)
    d = torch.from_numpy(dims.astype(np.int32)).to(dev)
    mw, mh = int(dims[:, 0].max()), int(dims[:, 1].max())
    lib = _lib.load()
    nbytes = ctypes.c_int64()
    _lib.check(lib.eca_nh_workspace_bytes(n, mw, mh, float(spacing), ctypes.byref(nbytes)),
               "eca_nh_workspace_bytes")
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    hd = torch.empty(n, dtype=torch.float64, device=dev)
    st = torch.empty(n, dtype=torch.int32, device=dev)
    _lib.check(lib.eca_area_hausdorff(_ptr(rp), _ptr(rt), _ptr(d), n, mw, mh, float(spacing), _ptr(ws),
                                      nbytes.value, _ptr(hd), _ptr(st), _stream(dev)),
               "eca_area_hausdorff")
    hd_h, st_h = hd.cpu().numpy(), st.cpu().numpy()
    for i in np.flatnonzero(st_h):
        if st_h[i] & 4:
            raise _lib.EcaError(f"eca_area_hausdorff: sample {i} exceeds the boundary bound")
        bad = as_circle(preds[i]) if st_h[i] & 1 else as_circle(truths[i])
        raise ValueError(f"{bad} does not intersect a {dims[i, 0]}x{dims[i, 1]} frame")
    # metrics.py:206-208, the scale in host FP64 (math.hypot) as the reference
    scale = np.array([REF_DIAGONAL / math.hypot(int(w), int(h)) for w, h in dims])
    return scale * hd_h


def area_error_px(predicted, truth, width: int, height: int, device=None) -> float:
    """Normalised Hausdorff distance between two content areas (metrics.py:211-223)."""
    return float(area_errors([predicted], [truth], (width, height), device=device)[0])


@dataclass(frozen=True, slots=True)
class SampleScore:
    sample_id: str
    nh_px: float
    label: MissClass


@dataclass(frozen=True, slots=True)
class EvalReport:
    """metrics.py:233-246: per-sample NH and the aggregate summary."""
    per_sample: tuple[SampleScore, ...]
    avg_error_px: float
    miss_pct: float
    bad_miss_pct: float


def evaluate_dataset(predictions: Mapping[str, ContentArea | Circle | None],
                     truths: Mapping[str, ContentArea | Circle | None],
                     frame_dims, device=None) -> EvalReport:
    """metrics.py:249-281 with every sample's NH from one batched GPU call."""
    missing = sorted(set(truths) ^ set(predictions))
    if missing:
        raise ValueError(f"sample ids do not align; unmatched: {missing[:20]}")
    if not predictions:
        raise ValueError("nothing to evaluate")
    ids = sorted(predictions)
    dims = [frame_dims[i] for i in ids] if isinstance(frame_dims, Mapping) else frame_dims
    nh = area_errors([predictions[i] for i in ids], [truths[i] for i in ids], dims, device=device)
    scores = [SampleScore(i, float(v), classify(float(v))) for i, v in zip(ids, nh)]
    n = len(scores)
    misses = sum(1 for s in scores if s.label is not MissClass.HIT)
    bad = sum(1 for s in scores if s.label is MissClass.BAD_MISS)
    return EvalReport(per_sample=tuple(scores),
                      avg_error_px=float(np.mean([s.nh_px for s in scores])),
                      miss_pct=100.0 * misses / n, bad_miss_pct=100.0 * bad / n)


def report_markdown(reports: Mapping[str, EvalReport]) -> str:
    """metrics.py:273-283."""
    lines = ["| Method | Avg. err. (px) | Miss (%) | Bad Miss (%) |", "| --- | --- | --- | --- |"]
    lines += [f"| {k} | {r.avg_error_px:.2f} | {r.miss_pct:.1f} | {r.bad_miss_pct:.1f} |"
              for k, r in reports.items()]
    return "\n".join(lines) + "\n"
