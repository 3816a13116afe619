"""Drop-in content-area API backed by the sm_100a kernels of libeca_b200.so.

Same names, argument meaning, result types and error behaviour as the
reference package's public surface (/root/reference/pkg/src/eca/__init__.py:10-65,
estimator.py:18-111, fitting.py:18-230, strips.py:13-77), plus the upstream
torch-content-area names the north star asks for (estimate_area, get_points,
fit_area, draw_mask, crop_area).

Inputs may be numpy arrays or torch tensors, HWC uint8, on the host or on a
CUDA device.  Host frames are not copied whole: only the strip rows the
kernels read cross PCIe (eca_h2d_bands).  Every computation runs on the GPU;
without a CUDA device these functions raise — there is no CPU fallback.
"""

from __future__ import annotations

import contextlib
import ctypes
import dataclasses
import functools
import inspect
import math
import threading
from dataclasses import dataclass
from enum import Enum
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from .params import EcaConfig, EcaParams, config_default
from .shapes import FULL_FRAME, Circle, CircularArea, ContentArea, EdgeCandidate, FullFrame, Side
from .stripnet import EdgeNet

WINDOW_ROWS = 7
HALF_WINDOW = 3
MIN_FRAME_WIDTH = 8
MIN_FRAME_HEIGHT = 2 * WINDOW_ROWS
MIN_CROP_SIDE = 14
MAX_FRAME_HEIGHT = 32767


# ----------------------------------------------------------------- types ---
@dataclass(frozen=True, slots=True)
class Handcrafted:
    """Edge scoring from gradient, centre-angle and preceding-intensity features."""


@dataclass(frozen=True, slots=True)
class Learned:
    """Edge scoring from the strip CNN (estimator.py:23-27)."""

    net: EdgeNet


EstimatorVariant = Handcrafted | Learned
HANDCRAFTED = Handcrafted()


class RejectionReason(Enum):
    NO_CANDIDATES = "no_candidates"
    LOW_SCORE = "low_score"
    GEOMETRY_GATE = "geometry_gate"


@dataclass(frozen=True, slots=True)
class Accepted:
    circle: Circle
    score: float
    inlier_count: int


@dataclass(frozen=True, slots=True)
class Rejected:
    reason: RejectionReason


FitResult = Accepted | Rejected


@dataclass(frozen=True, slots=True)
class StripScoreRow:
    """One strip's centre-row scores and its two half-row winners (handcrafted.py:25-31)."""

    scores: np.ndarray
    left_best: EdgeCandidate
    right_best: EdgeCandidate


@dataclass(frozen=True, slots=True)
class FrameError:
    """Per-index failure marker of a batch run (estimator.py:77-82)."""

    index: int
    message: str


_REASONS = {_lib.NO_CANDIDATES: RejectionReason.NO_CANDIDATES,
            _lib.LOW_SCORE: RejectionReason.LOW_SCORE,
            _lib.GEOMETRY_GATE: RejectionReason.GEOMETRY_GATE}


# ---------------------------------------------------------------- device ---
def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2210_14771_b200 runs on a CUDA device (B200, sm_100a); "
                           "no GPU is visible and there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"expected a CUDA device, got {d}")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _on(device) -> contextlib.AbstractContextManager:
    """Make ``device`` current for the native calls (they launch on the
    current device; torch tensors and streams may belong to another one)."""
    return torch.cuda.device(device)


def _with_device(fn):
    """Run ``fn`` with its ``device`` argument (default: the current device)
    made current.  Without a GPU ``fn`` runs as is (and raises where it needs one)."""
    sig = inspect.signature(fn)

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        if not torch.cuda.is_available():
            return fn(*args, **kwargs)
        with _on(_device(sig.bind(*args, **kwargs).arguments.get("device"))):
            return fn(*args, **kwargs)
    return wrapper


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _i32_array(vals) -> ctypes.Array:
    return (ctypes.c_int32 * max(1, len(vals)))(*vals)


# ---------------------------------------------------------------- frames ---
def validate_frame(frame) -> tuple[int, int]:
    """Shape / dtype check with the reference's messages (strips.py:13-27)."""
    if isinstance(frame, torch.Tensor):
        shape, ok_dtype, dtype = tuple(frame.shape), frame.dtype == torch.uint8, frame.dtype
    elif isinstance(frame, np.ndarray):
        shape, ok_dtype, dtype = frame.shape, frame.dtype == np.uint8, frame.dtype
    else:
        raise ValueError(f"expected an RGB frame of shape (H, W, 3), got {type(frame)}")
    if len(shape) != 3 or shape[2] != 3:
        raise ValueError(f"expected an RGB frame of shape (H, W, 3), got {shape}")
    if not ok_dtype:
        raise ValueError(f"expected uint8 pixel data, got {dtype}")
    height, width = shape[:2]
    if width < MIN_FRAME_WIDTH or height < MIN_FRAME_HEIGHT:
        raise ValueError(f"frame {width}x{height} too small: need width >= {MIN_FRAME_WIDTH} "
                         f"and height >= {MIN_FRAME_HEIGHT}")
    if width > _lib.MAX_WIDTH or height > MAX_FRAME_HEIGHT:
        # outside the kernels' envelope (the reference has no cap): a per-frame
        # ValueError, so estimate_batch reports a FrameError for this index
        raise ValueError(f"frame {width}x{height} too large: the GPU kernels take width <= "
                         f"{_lib.MAX_WIDTH} and height <= {MAX_FRAME_HEIGHT}")
    return width, height


def _check_config(cfg: EcaConfig) -> None:
    """The native limits on EcaConfig (include/eca_b200.h) as ValueError."""
    if cfg.strip_count > _lib.MAX_STRIPS:
        raise ValueError(f"strip_count {cfg.strip_count} exceeds the GPU limit {_lib.MAX_STRIPS}")
    if cfg.ransac_attempts > _lib.MAX_ATTEMPTS:
        raise ValueError(f"ransac_attempts {cfg.ransac_attempts} exceeds the GPU limit "
                         f"{_lib.MAX_ATTEMPTS}")


@lru_cache(maxsize=256)
def _strip_rows(height: int, count: int, weighting: float) -> tuple[int, ...]:
    buf = (ctypes.c_int32 * count)()
    n = _lib.check(_lib.load().eca_strip_rows(height, count, weighting, buf), "eca_strip_rows")
    return tuple(buf[:n])


def strip_heights(height: int, count: int, weighting: float) -> list[int]:
    """Sigmoid strip centre rows, rounded, clamped, de-duplicated (strips.py:41-60)."""
    if height < MIN_FRAME_HEIGHT:
        raise ValueError(f"height {height} cannot host a {WINDOW_ROWS}-row window")
    if count < 2:
        raise ValueError(f"need at least 2 strips, got {count}")
    if weighting <= 0:
        raise ValueError(f"weighting must be positive, got {weighting}")
    return list(_strip_rows(int(height), int(count), float(weighting)))


@dataclass
class _DevFrames:
    """A batch of same-size frames as the kernels see it."""

    ptr: ctypes.c_void_p
    batch: int
    fstride: int
    rstride: int
    band: ctypes.Array | None     # memory row of each strip's first band row, or None
    keep: object                  # owner of the device memory


def _to_device_frames(frames, rows, half: int, device) -> _DevFrames:
    """Place a batch on the GPU.  CUDA tensors are used in place; host frames
    ship only rows [y-half, y+half] of every strip (eca_h2d_bands)."""
    if isinstance(frames, (list, tuple)):
        if all(isinstance(f, torch.Tensor) and f.is_cuda for f in frames):
            frames = torch.stack([f.to(device) for f in frames])
        else:
            return _host_bands([np.asarray(f) if not isinstance(f, torch.Tensor) else f
                                for f in frames], rows, half, device)
    if isinstance(frames, torch.Tensor) and frames.is_cuda:
        t = frames.to(device)
        if t.dim() == 3:
            t = t.unsqueeze(0)
        if t.stride(3) != 1 or t.stride(2) != 3:
            t = t.contiguous()
        return _DevFrames(_ptr(t), t.shape[0], t.stride(0), t.stride(1), None, t)
    return _host_bands([frames], rows, half, device)


def _host_bands(items, rows, half: int, device) -> _DevFrames:
    """items: list of host arrays/tensors, each (H,W,3) or (B,H,W,3)."""
    lib = _lib.load()
    first = _i32_array([r - half for r in rows])
    nb, rpb = len(rows), 2 * half + 1
    total = 0
    views = []
    for it in items:
        a = it.numpy() if isinstance(it, torch.Tensor) else it
        if a.ndim == 3:
            a = a[None]
        # packed pixels, and non-negative row / frame strides (e.g. frame[::-1])
        if a.strides[-1] != 1 or a.strides[-2] != 3 or a.strides[1] < 3 * a.shape[2] or a.strides[0] < 0:
            a = np.ascontiguousarray(a)
        views.append(a)
        total += a.shape[0]
    h, w = views[0].shape[1:3]
    out = torch.empty((total, nb * rpb, w, 3), dtype=torch.uint8, device=device)
    stream = _stream(device)
    off = 0
    for a in views:
        rc = lib.eca_h2d_bands(ctypes.c_void_p(a.ctypes.data), a.shape[0], a.strides[0], a.strides[1],
                               first, nb, rpb, w, ctypes.c_void_p(out[off].data_ptr()), stream)
        _lib.check(rc, "eca_h2d_bands")
        off += a.shape[0]
    band = _i32_array([k * rpb for k in range(nb)])
    # pageable sources are staged before cudaMemcpy2DAsync returns; pinned
    # sources belong to the caller, who keeps them alive
    return _DevFrames(_ptr(out), total, out.stride(0), out.stride(1), band, (out, views))


# -------------------------------------------------------------- triplets ---
_TRIPLETS: dict = {}


def triplet_table(seed: int, attempts: int, max_n: int) -> np.ndarray:
    """Seeded hypotheses for every candidate count n in [3, max_n]
    (fitting.py:147-156), shape (max_n-2, attempts, 3) int16."""
    if seed < 0:
        raise ValueError("expected non-negative integer seed")
    max_n = max(3, max_n)
    out = np.empty((max_n - 2, attempts, 3), dtype=np.int16)
    rc = _lib.load().eca_triplet_table(int(seed), attempts, max_n,
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_int16)))
    _lib.check(rc, "eca_triplet_table")
    return out


def _dev_triplets(seed: int, attempts: int, max_n: int, device) -> torch.Tensor:
    key = (int(seed), attempts, max(3, max_n), str(device))
    t = _TRIPLETS.get(key)
    if t is None:
        t = torch.from_numpy(triplet_table(seed, attempts, max_n)).to(device)
        if len(_TRIPLETS) > 64:
            _TRIPLETS.clear()
        _TRIPLETS[key] = t
    return t


_WORKSPACES: dict = {}


def _stream_key(device) -> tuple:
    return (str(device), torch.cuda.current_stream(device).cuda_stream)


def points_workspace(batch: int, n_strips: int, device) -> torch.Tensor:
    """Device scratch for eca_points_handcrafted (tickets + survivor slots),
    zero-initialised once (the kernels leave the tickets zeroed), cached per
    (device, current stream): calls on different streams never share one."""
    n = ctypes.c_int64()
    _lib.check(_lib.load().eca_points_workspace_bytes(batch, n_strips, ctypes.byref(n)),
               "eca_points_workspace_bytes")
    key = _stream_key(device)
    t = _WORKSPACES.get(key)
    if t is None or t.numel() < n.value:
        t = torch.zeros(max(n.value, 1 << 20), dtype=torch.uint8, device=device)
        _WORKSPACES[key] = t
    return t


_COUNTERS: dict = {}


def _dev_counters(n: int, device) -> torch.Tensor:
    """Per-frame completion counters of the fused launch (left zeroed), cached
    per (device, current stream)."""
    key = _stream_key(device)
    t = _COUNTERS.get(key)
    if t is None or t.numel() < n:
        t = torch.zeros(max(n, 1024), dtype=torch.int32, device=device)
        _COUNTERS[key] = t
    return t


# --------------------------------------------------------------- records ---
def _records_to_results(rec: torch.Tensor) -> list[ContentArea]:
    """(B,5) float64 EcaFitRecord rows -> CircularArea | FULL_FRAME."""
    r = rec.detach().cpu().numpy()
    status = r.view(np.int32).reshape(len(r), 10)[:, 9]
    out = []
    for i in range(len(r)):
        if status[i] == _lib.ACCEPTED:
            out.append(CircularArea(Circle(float(r[i, 0]), float(r[i, 1]), float(r[i, 2])),
                                    float(r[i, 3])))
        else:
            out.append(FULL_FRAME)
    return out


def _record_to_fit(row: np.ndarray) -> FitResult:
    i32 = row.view(np.int32)
    status, inl = int(i32[9]), int(i32[8])
    if status == _lib.ACCEPTED:
        return Accepted(Circle(float(row[0]), float(row[1]), float(row[2])), float(row[3]), inl)
    return Rejected(_REASONS[status])


def records_to_fits(rec: torch.Tensor) -> list[FitResult]:
    r = rec.detach().cpu().numpy()
    return [_record_to_fit(r[i]) for i in range(len(r))]


# ------------------------------------------------------------- batch core ---
def _handcrafted_batch(df: _DevFrames, width: int, height: int, rows, cfg: EcaConfig, seed: int,
                       device, center=None):
    """One fused launch: strip scoring -> candidates -> filter -> RANSAC."""
    lib = _lib.load()
    s = len(rows)
    b = df.batch
    xs = torch.empty((b, 2 * s), dtype=torch.int32, device=device)
    ys = torch.empty_like(xs)
    sc = torch.empty((b, 2 * s), dtype=torch.float64, device=device)
    rec = torch.empty((b, 5), dtype=torch.float64, device=device)
    params = cfg.device_params(width, height, center)
    trip = _dev_triplets(seed, cfg.ransac_attempts, 2 * s, device)
    if b <= 16:   # latency: one fused launch
        cnt = _dev_counters(b, device)
        rc = lib.eca_estimate_handcrafted(df.ptr, b, df.fstride, df.rstride, _i32_array(rows),
                                          df.band, s, ctypes.byref(params), _ptr(trip), _ptr(cnt),
                                          _ptr(xs), _ptr(ys), _ptr(sc), _ptr(rec), _stream(device))
        _lib.check(rc, "eca_estimate_handcrafted")
        return xs, ys, sc, rec
    # throughput: strip kernel, then the fit kernel (one warp per frame)
    ws = points_workspace(b, s, device)
    rc = lib.eca_points_handcrafted(df.ptr, b, df.fstride, df.rstride, _i32_array(rows), df.band, s,
                                    ctypes.byref(params), _ptr(xs), _ptr(ys), _ptr(sc), _ptr(ws),
                                    _stream(device))
    _lib.check(rc, "eca_points_handcrafted")
    rc = lib.eca_fit(_ptr(xs), _ptr(ys), _ptr(sc), b, 2 * s, ctypes.byref(params), _ptr(trip), 0,
                     _ptr(rec), _stream(device))
    _lib.check(rc, "eca_fit")
    return xs, ys, sc, rec


def _learned_points(df: _DevFrames, width: int, height: int, rows, net: EdgeNet, device):
    lib = _lib.load()
    s = len(rows)
    b = df.batch
    w_dev, norm = _dev_net(net, device)
    xs = torch.empty((b, 2 * s), dtype=torch.int32, device=device)
    ys = torch.empty_like(xs)
    sc = torch.empty((b, 2 * s), dtype=torch.float64, device=device)
    probs = torch.empty((b, s, width - 6), dtype=torch.float32, device=device)
    for b0 in range(0, b, 65535):
        nb = min(65535, b - b0)
        rc = lib.eca_points_learned(ctypes.c_void_p(df.ptr.value + b0 * df.fstride), nb, df.fstride,
                                    df.rstride, _i32_array(rows), df.band, s, height, width,
                                    _ptr(w_dev), norm, _ptr(probs[b0:]), _ptr(xs[b0:]),
                                    _ptr(ys[b0:]), _ptr(sc[b0:]), _stream(device))
        _lib.check(rc, "eca_points_learned")
    return xs, ys, sc, probs


_NETS: dict = {}


def _dev_net(net: EdgeNet, device):
    key = (id(net), str(device))
    packed = net.packed()
    hit = _NETS.get(key)
    if hit is None or not np.array_equal(hit[2], packed):
        w = torch.from_numpy(packed).to(device)
        norm = (ctypes.c_double * 6)(*net.norm_array())
        hit = (w, norm, packed)
        _NETS[key] = hit
    return hit[0], hit[1]


def _fit_batch(xs, ys, sc, width, height, cfg: EcaConfig, seed: int, device, *, exhaustive=False,
               center=None, prefiltered=False) -> torch.Tensor:
    lib = _lib.load()
    b, n = xs.shape
    params = cfg.device_params(width, height, center)
    if prefiltered:        # ransac_fit receives already-filtered candidates
        params.edge_margin_px = -(2 ** 30)
        params.min_point_score = -math.inf
    trip = _dev_triplets(seed, cfg.ransac_attempts, n, device)
    rec = torch.empty((b, 5), dtype=torch.float64, device=device)
    rc = lib.eca_fit(_ptr(xs), _ptr(ys), _ptr(sc), b, n, ctypes.byref(params), _ptr(trip),
                     1 if exhaustive else 0, _ptr(rec), _stream(device))
    _lib.check(rc, "eca_fit")
    return rec


def _candidates(xs_row, ys_row, sc_row, s) -> list[EdgeCandidate]:
    return ([EdgeCandidate(int(xs_row[k]), int(ys_row[k]), float(sc_row[k]), Side.LEFT)
             for k in range(s)] +
            [EdgeCandidate(int(xs_row[s + k]), int(ys_row[s + k]), float(sc_row[s + k]), Side.RIGHT)
             for k in range(s)])


# ------------------------------------------------------------ public API ---
@_with_device
def score_frame_strips(frame, variant: EstimatorVariant = HANDCRAFTED, cfg: EcaConfig | None = None,
                       device=None):
    """Scored strip rows for one frame (estimator.py:35-52): (rows, (W, H))."""
    cfg = cfg or config_default()
    width, height = validate_frame(frame)
    rows = strip_heights(height, cfg.strip_count, cfg.strip_weighting)
    dev = _device(device)
    s = len(rows)
    if isinstance(variant, Learned):
        df = _to_device_frames(frame, rows, HALF_WINDOW, dev)
        xs, ys, sc, probs = _learned_points(df, width, height, rows, variant.net, dev)
        scores = np.zeros((s, width), dtype=np.float64)
        scores[:, HALF_WINDOW:width - HALF_WINDOW] = probs[0].cpu().numpy()
    else:
        df = _to_device_frames(frame, rows, 1, dev)
        lib = _lib.load()
        out = torch.empty((1, s, width), dtype=torch.float64, device=dev)
        xs = torch.empty((1, 2 * s), dtype=torch.int32, device=dev)
        ys = torch.empty_like(xs)
        sc = torch.empty((1, 2 * s), dtype=torch.float64, device=dev)
        rc = lib.eca_score_rows_handcrafted(df.ptr, 1, df.fstride, df.rstride, _i32_array(rows),
                                            df.band, s, ctypes.byref(cfg.device_params(width, height)),
                                            _ptr(out), _ptr(xs), _ptr(ys), _ptr(sc), _stream(dev))
        _lib.check(rc, "eca_score_rows_handcrafted")
        scores = out[0].cpu().numpy()
    c = _candidates(xs[0].cpu().numpy(), ys[0].cpu().numpy(), sc[0].cpu().numpy(), s)
    return [StripScoreRow(scores[k], c[k], c[s + k]) for k in range(s)], (width, height)


def get_points(frame, variant: EstimatorVariant = HANDCRAFTED, cfg: EcaConfig | None = None,
               device=None) -> list[EdgeCandidate]:
    """North-star name: every half-strip winner, lefts then rights (estimator.py:69)."""
    return get_points_batch([frame], variant, cfg, device)[0]


@_with_device
def get_points_batch(frames, variant: EstimatorVariant = HANDCRAFTED, cfg: EcaConfig | None = None,
                     device=None) -> list[list[EdgeCandidate]]:
    cfg = cfg or config_default()
    dev = _device(device)
    width, height = _batch_shape(frames)
    rows = strip_heights(height, cfg.strip_count, cfg.strip_weighting)
    s = len(rows)
    if isinstance(variant, Learned):
        df = _to_device_frames(frames, rows, HALF_WINDOW, dev)
        xs, ys, sc, _ = _learned_points(df, width, height, rows, variant.net, dev)
    else:
        df = _to_device_frames(frames, rows, 1, dev)
        lib = _lib.load()
        xs = torch.empty((df.batch, 2 * s), dtype=torch.int32, device=dev)
        ys = torch.empty_like(xs)
        sc = torch.empty((df.batch, 2 * s), dtype=torch.float64, device=dev)
        ws = points_workspace(df.batch, s, dev)
        rc = lib.eca_points_handcrafted(df.ptr, df.batch, df.fstride, df.rstride, _i32_array(rows),
                                        df.band, s, ctypes.byref(cfg.device_params(width, height)),
                                        _ptr(xs), _ptr(ys), _ptr(sc), _ptr(ws), _stream(dev))
        _lib.check(rc, "eca_points_handcrafted")
    xs, ys, sc = xs.cpu().numpy(), ys.cpu().numpy(), sc.cpu().numpy()
    return [_candidates(xs[i], ys[i], sc[i], s) for i in range(len(xs))]


def filter_candidates(candidates: list[EdgeCandidate], frame_size: tuple[int, int],
                      cfg: EcaConfig) -> list[EdgeCandidate]:
    """Order-preserving margin + score filter (fitting.py:39-52).  The batched
    device path applies the same rule inside the fitter kernel."""
    width, height = frame_size
    m = cfg.edge_margin_px
    return [c for c in candidates
            if min(c.x, width - 1 - c.x, c.y, height - 1 - c.y) >= m and c.score >= cfg.min_point_score]


@_with_device
def ransac_fit(candidates: list[EdgeCandidate], frame_size: tuple[int, int], cfg: EcaConfig,
               seed: int = 0, *, exhaustive: bool = False,
               center: tuple[float, float] | None = None, device=None) -> FitResult:
    """Seeded RANSAC + iterated least squares on the GPU (fitting.py:159-230)."""
    n = len(candidates)
    if n < 3:
        return Rejected(RejectionReason.NO_CANDIDATES)
    if n > 2 * _lib.MAX_STRIPS:
        raise ValueError(f"at most {2 * _lib.MAX_STRIPS} candidates per fit, got {n}")
    dev = _device(device)
    width, height = frame_size
    xs = torch.tensor([[int(c.x) for c in candidates]], dtype=torch.int32).to(dev)
    ys = torch.tensor([[int(c.y) for c in candidates]], dtype=torch.int32).to(dev)
    sc = torch.tensor([[float(c.score) for c in candidates]], dtype=torch.float64).to(dev)
    rec = _fit_batch(xs, ys, sc, width, height, cfg, seed, dev, exhaustive=exhaustive,
                     center=center, prefiltered=True)
    return _record_to_fit(rec[0].cpu().numpy())


@_with_device
def fit_area(candidates: list[EdgeCandidate], frame_size: tuple[int, int],
             cfg: EcaConfig | None = None, seed: int = 0, device=None) -> FitResult:
    """North-star name: filter_candidates + ransac_fit in one device call."""
    cfg = cfg or config_default()
    n = len(candidates)
    if n == 0:
        return Rejected(RejectionReason.NO_CANDIDATES)
    if n > 2 * _lib.MAX_STRIPS:
        raise ValueError(f"at most {2 * _lib.MAX_STRIPS} candidates per fit, got {n}")
    dev = _device(device)
    width, height = frame_size
    xs = torch.tensor([[int(c.x) for c in candidates]], dtype=torch.int32).to(dev)
    ys = torch.tensor([[int(c.y) for c in candidates]], dtype=torch.int32).to(dev)
    sc = torch.tensor([[float(c.score) for c in candidates]], dtype=torch.float64).to(dev)
    return _record_to_fit(_fit_batch(xs, ys, sc, width, height, cfg, seed, dev)[0].cpu().numpy())


def _batch_shape(frames) -> tuple[int, int]:
    if isinstance(frames, (list, tuple)):
        if not frames:
            raise ValueError("empty batch")
        sizes = {validate_frame(f) for f in frames}
        if len(sizes) != 1:
            raise ValueError(f"frames of one batch must share a size, got {sorted(sizes)}")
        return sizes.pop()
    if frames.ndim == 4:
        return validate_frame(frames[0])
    return validate_frame(frames)


class _FrameEstimator:
    """estimate() of ONE handcrafted frame of a fixed (H, W, cfg, seed, device),
    everything preallocated: one fused launch (strip scoring -> candidates ->
    filter -> RANSAC, eca_estimate_handcrafted) whose fit writes the record
    straight into pinned host memory, status word last; the host polls that
    word (a bounded spin, then a stream synchronisation that also raises any
    kernel error) instead of waking from a synchronisation.  Host
    frames: the 3 rows of every strip are copied into a pinned buffer that the
    kernel reads over PCIe (no H2D copy, no full-frame transfer).  A lock
    serialises callers (the buffers are shared)."""

    def __init__(self, height: int, width: int, cfg: EcaConfig, seed: int, device):
        self.h, self.w, self.dev = height, width, device
        self.rows = strip_heights(height, cfg.strip_count, cfg.strip_weighting)
        s = self.s = len(self.rows)
        self.c_rows = _i32_array(self.rows)
        self.c_band = _i32_array([3 * k for k in range(s)])
        self.params = cfg.device_params(width, height)
        self.p_params = ctypes.byref(self.params)
        with _on(device):
            self.trip = _dev_triplets(seed, cfg.ransac_attempts, 2 * s, device)
            self.cnt = torch.zeros(64, dtype=torch.int32, device=device)
            self.xs = torch.empty((1, 2 * s), dtype=torch.int32, device=device)
            self.ys = torch.empty_like(self.xs)
            self.sc = torch.empty((1, 2 * s), dtype=torch.float64, device=device)
        self.rec_host = torch.zeros((1, 5), dtype=torch.float64).pin_memory()
        self.rec_np = self.rec_host.numpy()
        self.rec_i32 = self.rec_np.view(np.int32).reshape(-1)   # [9]: the status word
        self.bands_host = torch.empty((3 * s, width, 3), dtype=torch.uint8).pin_memory()
        self.bands_np = self.bands_host.numpy()
        self.row_idx = np.array([r + d for r in self.rows for d in (-1, 0, 1)], dtype=np.intp)
        self.args = [_ptr(self.trip), _ptr(self.cnt), _ptr(self.xs), _ptr(self.ys), _ptr(self.sc),
                     ctypes.c_void_p(self.rec_host.data_ptr())]
        self.fn = _lib.load().eca_estimate_handcrafted
        self.lock = threading.Lock()

    def __call__(self, frame) -> ContentArea:
        if torch.cuda.current_device() == self.dev.index:   # (the device switch costs microseconds)
            with self.lock:
                return self._run(frame)
        with self.lock, _on(self.dev):
            return self._run(frame)

    def _run(self, frame) -> ContentArea:
        if isinstance(frame, torch.Tensor) and frame.is_cuda:
            t = frame if frame.device == self.dev else frame.to(self.dev)
            if t.stride(2) != 1 or t.stride(1) != 3 or t.stride(0) < 3 * self.w:
                t = t.contiguous()
            ptr, rs, band = ctypes.c_void_p(t.data_ptr()), t.stride(0), None
        else:
            a = frame.numpy() if isinstance(frame, torch.Tensor) else frame
            np.take(a, self.row_idx, axis=0, out=self.bands_np)
            ptr, rs, band = ctypes.c_void_p(self.bands_host.data_ptr()), 3 * self.w, self.c_band
        raw = _raw_stream(self.dev)
        st32 = self.rec_i32
        st32[9] = _PENDING
        _lib.check(self.fn(ptr, 1, 0, rs, self.c_rows, band, self.s, self.p_params, *self.args,
                           ctypes.c_void_p(raw)), "eca_estimate_handcrafted")
        spins = 0
        while st32[9] == _PENDING:
            spins += 1
            if spins & 0x3FF == 0 and spins > _SPIN_LIMIT:
                torch.cuda.current_stream(self.dev).synchronize()   # raises a kernel error
                if st32[9] == _PENDING:
                    raise _lib.EcaError("eca_estimate_handcrafted: the record was not written")
        r = self.rec_np[0]
        if int(st32[9]) == _lib.ACCEPTED:
            return CircularArea(Circle(float(r[0]), float(r[1]), float(r[2])), float(r[3]))
        return FULL_FRAME


_PENDING = -0x7FFFFFFF        # a status value outside EcaStatus: "not written yet"
_SPIN_LIMIT = 1 << 16          # polls of the status word before a stream synchronisation
try:                           # the current stream's raw handle without a Stream object
    _RAW_STREAM = torch._C._cuda_getCurrentRawStream
except AttributeError:         # pragma: no cover
    _RAW_STREAM = None


def _raw_stream(dev: torch.device) -> int:
    if _RAW_STREAM is not None:
        return _RAW_STREAM(dev.index)
    return torch.cuda.current_stream(dev).cuda_stream


_FRAME_ESTIMATORS: dict = {}


def estimate(frame, variant: EstimatorVariant = HANDCRAFTED, cfg: EcaConfig | None = None,
             seed: int = 0, device=None) -> ContentArea:
    """Content area of one RGB frame (estimator.py:55-74).  The handcrafted
    variant takes the cached single-frame path (_FrameEstimator)."""
    width, height = validate_frame(frame)
    cfg = cfg or config_default()
    if isinstance(variant, Learned):
        out = estimate_batch([frame], variant, cfg, seed, device=device)[0]
        if isinstance(out, FrameError):
            raise ValueError(out.message)
        return out
    if seed < 0:
        raise ValueError("expected non-negative integer seed")
    _check_config(cfg)
    if device is None:   # the frame's device, else the current one
        if isinstance(frame, torch.Tensor) and frame.is_cuda:
            device = frame.device.index
        else:
            if not torch.cuda.is_available():
                _device(None)   # raises: no GPU, no CPU fallback
            device = torch.cuda.current_device()
    key = (height, width, cfg, seed, device)
    est = _FRAME_ESTIMATORS.get(key)
    if est is None:
        dev = _device(device if not isinstance(device, int) else torch.device("cuda", device))
        if len(_FRAME_ESTIMATORS) > 32:
            _FRAME_ESTIMATORS.clear()
        est = _FRAME_ESTIMATORS[key] = _FrameEstimator(height, width, cfg, seed, dev)
    return est(frame)


estimate_area = estimate


def estimate_batch(frames, variant: EstimatorVariant = HANDCRAFTED, cfg: EcaConfig | None = None,
                   seed: int = 0, threads: int | None = None, device=None) -> list[ContentArea | FrameError]:
    """Order-preserving batch; malformed frames become FrameError (estimator.py:85-111).

    Frames are grouped by size and each group runs as one batched launch;
    ``threads`` is accepted for signature compatibility (the GPU replaces the
    reference's thread pool)."""
    cfg = cfg or config_default()
    _check_config(cfg)
    items = list(frames) if not (isinstance(frames, (np.ndarray, torch.Tensor)) and frames.ndim == 4) \
        else [frames[i] for i in range(frames.shape[0])]
    out: list = [None] * len(items)
    groups: dict = {}
    for i, f in enumerate(items):
        try:
            w, h = validate_frame(f)
            rows = strip_heights(h, cfg.strip_count, cfg.strip_weighting)
        except ValueError as exc:
            out[i] = FrameError(i, str(exc))
            continue
        groups.setdefault((w, h), []).append(i)
    if not groups:
        return out
    dev = _device(device)
    with _on(dev):
        for (w, h), idx in groups.items():
            rows = strip_heights(h, cfg.strip_count, cfg.strip_weighting)
            sub = [items[i] for i in idx]
            rec = _estimate_group(sub, w, h, rows, variant, cfg, seed, dev)
            for i, res in zip(idx, _records_to_results(rec)):
                out[i] = res
    return out


def _estimate_group(sub, w, h, rows, variant, cfg, seed, dev) -> torch.Tensor:
    if isinstance(variant, Learned):
        df = _to_device_frames(sub, rows, HALF_WINDOW, dev)
        xs, ys, sc, _ = _learned_points(df, w, h, rows, variant.net, dev)
        return _fit_batch(xs, ys, sc, w, h, cfg, seed, dev)
    df = _to_device_frames(sub, rows, 1, dev)
    return _handcrafted_batch(df, w, h, rows, cfg, seed, dev)[3]


# ------------------------------------------------------------- mask / crop ---
def _area_records(areas, device) -> torch.Tensor:
    rec = np.zeros((len(areas), 5), dtype=np.float64)
    i32 = rec.view(np.int32).reshape(len(areas), 10)
    for i, a in enumerate(areas):
        if isinstance(a, CircularArea):
            a = a.circle
        if isinstance(a, Circle):
            rec[i, :3] = (a.cx, a.cy, a.r)
            i32[i, 9] = _lib.ACCEPTED
        elif isinstance(a, FullFrame) or a is None:
            i32[i, 9] = _lib.LOW_SCORE
        else:
            raise TypeError(f"expected CircularArea, Circle or FullFrame, got {type(a)}")
    return torch.from_numpy(rec).to(device)


@_with_device
def draw_mask(areas, height: int, width: int, device=None) -> torch.Tensor:
    """uint8 content masks on the GPU: 1 inside the closed disk at pixel centres
    (geometry.py:30-34), all ones for FullFrame.  ``areas`` is one area (-> (H,W))
    or a list / an (B,5) record tensor (-> (B,H,W))."""
    dev = _device(device)
    single = not isinstance(areas, (list, tuple, torch.Tensor))
    if isinstance(areas, torch.Tensor):
        rec = areas.to(dev, dtype=torch.float64).contiguous()
    else:
        rec = _area_records([areas] if single else list(areas), dev)
    b = rec.shape[0]
    out = torch.empty((b, height, width), dtype=torch.uint8, device=dev)
    rc = _lib.load().eca_draw_mask(_ptr(rec), b, height, width, _ptr(out), height * width, _stream(dev))
    _lib.check(rc, "eca_draw_mask")
    return out[0] if single else out


@_with_device
def crop_bounds(areas, height: int, width: int, device=None) -> list[tuple[int, int, int, int] | None]:
    """crop_augment's inclusive rectangle per area (dataset.py:151-187), or None."""
    dev = _device(device)
    rec = _area_records(list(areas), dev)
    out = torch.empty((len(areas), 4), dtype=torch.int32, device=dev)
    rc = _lib.load().eca_crop_bounds(_ptr(rec), len(areas), height, width, _ptr(out), _stream(dev))
    _lib.check(rc, "eca_crop_bounds")
    return [None if r[0] < 0 else tuple(int(v) for v in r) for r in out.cpu().numpy()]


@_with_device
def crop_area(frame, area, device=None):
    """Largest centred axis-aligned rectangle inside the content disk, copied out
    on the GPU (dataset.py:151-187).  FullFrame raises ValueError like the
    reference; returns None where the reference does."""
    if not isinstance(area, (CircularArea, Circle)):
        raise ValueError("crop augmentation requires a circular annotation")
    width, height = _frame_wh(frame)
    dev = _device(device)
    rec = _area_records([area], dev)
    bounds = torch.empty((1, 4), dtype=torch.int32, device=dev)
    lib = _lib.load()
    _lib.check(lib.eca_crop_bounds(_ptr(rec), 1, height, width, _ptr(bounds), _stream(dev)),
               "eca_crop_bounds")
    x0, y0, x1, y1 = (int(v) for v in bounds[0].cpu())
    if x0 < 0:
        return None
    src = frame if isinstance(frame, torch.Tensor) and frame.is_cuda else \
        torch.as_tensor(np.ascontiguousarray(frame)).to(dev)
    if src.stride(2) != 1 or src.stride(1) != 3:
        src = src.contiguous()
    out = torch.empty((y1 - y0 + 1, x1 - x0 + 1, 3), dtype=torch.uint8, device=dev)
    offs = torch.zeros(1, dtype=torch.int64, device=dev)
    rc = lib.eca_crop_copy(_ptr(src), 1, src.numel(), src.stride(0), _ptr(bounds), _ptr(offs),
                           _ptr(out), y1 - y0 + 1, _stream(dev))
    _lib.check(rc, "eca_crop_copy")
    return out


def _frame_wh(frame) -> tuple[int, int]:
    shape = tuple(frame.shape)
    return shape[1], shape[0]


def crop_augment(annotation, frame):
    """Reference-shaped wrapper (dataset.py:151-187): ``annotation.area`` is the
    circle; returns (crop, annotation with area=None and "_crop" id) or None.
    The crop comes back as the input's array type."""
    circle = getattr(annotation, "area", annotation)
    if circle is None or isinstance(circle, FullFrame):
        raise ValueError("crop augmentation requires a circular annotation")
    crop = crop_area(frame, circle)
    if crop is None:
        return None
    if isinstance(frame, np.ndarray):
        crop = crop.cpu().numpy()
    if dataclasses.is_dataclass(annotation) and hasattr(annotation, "sample_id"):
        annotation = dataclasses.replace(annotation, sample_id=annotation.sample_id + "_crop",
                                         area=None, image_path="")
    return crop, annotation
