"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the content-area hot path of the reference package
(`/root/reference/pkg/src/eca`, import name ``eca``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The shipped package (``paper_2210_14771_b200``) never
imports it and has no CPU fallback.

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the reference
itself (in the build container, where ``/root/reference`` exists) and writes
its outputs as fixtures; ``tests/test_oracle_golden.py`` asserts this module
reproduces every fixture (strip rows, per-column scores, candidates, triplets,
fits, learned probabilities, masks, crop bounds) bit-for-bit.

Each function cites the reference file:line it restates.  Arithmetic is kept
in the reference's evaluation order (numpy ufuncs, no fused multiply-add) so
the results are identical bits on the same host.

Config objects: any object exposing the ``EcaConfig`` field names
(config.py:14-60) works, e.g. ``paper_2210_14771_b200.EcaConfig``.
"""

from __future__ import annotations

import math
from itertools import combinations

import numpy as np

HALF = 3          # strips.py:8  (7-row window, centre +/- 3)
MIN_W, MIN_H = 8, 14   # strips.py:9-10
MIN_CROP = 14     # dataset.py:34

# status codes shared with the CUDA fitter (include/eca_b200.h)
ACCEPTED, NO_CANDIDATES, LOW_SCORE, GEOMETRY_GATE = 0, 1, 2, 3


# ----------------------------------------------------------------------------
# strip placement                                           strips.py:30-60
# ----------------------------------------------------------------------------
def strip_rows(height: int, count: int, weighting: float) -> list[int]:
    """Sigmoid strip centres, round half-up, clamp, drop consecutive repeats."""
    idx = np.arange(count, dtype=np.float64)
    raw = height / (1.0 + np.exp(-(weighting / count) * (idx - (count - 1) / 2.0)))
    rows = np.clip(np.floor(raw + 0.5).astype(np.int64), HALF, height - HALF - 1)
    keep = np.ones(len(rows), dtype=bool)
    keep[1:] = rows[1:] != rows[:-1]
    return [int(v) for v in rows[keep]]


# ----------------------------------------------------------------------------
# handcrafted scoring                              handcrafted.py:148-205, 120-138
# ----------------------------------------------------------------------------
def score_rows(frame: np.ndarray, rows: list[int], cfg) -> np.ndarray:
    """(S, W) float64 edge scores of each strip's centre row."""
    height, width = frame.shape[:2]
    r = np.asarray(rows, dtype=np.int64)
    # only rows h-1, h, h+1 carry signal (handcrafted.py:164-169)
    band = frame[r[:, None] + np.arange(-1, 2)[None, :]]          # (S,3,W,3) u8
    g = (band[..., 0].astype(np.uint16) + band[..., 1] + band[..., 2]) / 3.0
    lo, mi, hi = g[..., :-2], g[..., 1:-1], g[..., 2:]
    gx = np.zeros((len(rows), width))
    gy = np.zeros((len(rows), width))
    # association order of handcrafted.py:47-52 (exact mirror symmetry)
    gx[:, 1:-1] = (hi[:, 0] - lo[:, 0]) + 2.0 * (hi[:, 1] - lo[:, 1]) + (hi[:, 2] - lo[:, 2])
    gy[:, 1:-1] = ((lo[:, 2] + hi[:, 2]) + 2.0 * mi[:, 2]) - ((lo[:, 0] + hi[:, 0]) + 2.0 * mi[:, 0])
    centre = g[:, 1, :]

    cx, cy = (width - 1) / 2.0, (height - 1) / 2.0                # geometry.py:37-44
    tox = cx - np.arange(width, dtype=np.float64)[None, :]
    toy = cy - r.astype(np.float64)[:, None]
    k = 180.0 / (math.pi * cfg.angle_threshold_deg)
    ang = np.arctan2(np.abs(gx * toy - gy * tox), gx * tox + gy * toy) * k
    ang[(gx == 0.0) & (gy == 0.0)] = math.pi * k

    # preceding max, border -> column, column excluded (handcrafted.py:184-191)
    split = (width + 1) // 2
    prec = np.zeros_like(centre)
    prec[:, 1:] = np.maximum.accumulate(centre[:, :-1], axis=1)
    suffix = np.maximum.accumulate(centre[:, ::-1], axis=1)[:, ::-1]
    prec[:, split:] = 0.0
    prec[:, split:-1] = suffix[:, split + 1:]

    s = (
        np.tanh(np.sqrt(gx * gx + gy * gy) / cfg.gradient_threshold)
        * (2.0 / (1.0 + np.exp(2.0 * ang)))
        * (2.0 / (1.0 + np.exp(2.0 * prec / cfg.intensity_threshold)))
    )
    s[:, 0] = 0.0
    s[:, -1] = 0.0
    return s


def pick_halves(scores: np.ndarray):
    """Per row: (left x, right x).  Left ties -> smallest x, right -> largest."""
    width = scores.shape[1]
    split = (width + 1) // 2
    lx = np.argmax(scores[:, :split], axis=1)
    rx = width - 1 - np.argmax(scores[:, split:][:, ::-1], axis=1)
    return lx, rx


def candidates_from_scores(scores: np.ndarray, rows: list[int]):
    """Flatten in estimator.py:69 order: every left winner, then every right.

    Returns (x int64[2S], y int64[2S], score float64[2S])."""
    lx, rx = pick_halves(scores)
    k = np.arange(len(rows))
    xs = np.concatenate([lx, rx]).astype(np.int64)
    ys = np.concatenate([rows, rows]).astype(np.int64)
    sc = np.concatenate([scores[k, lx], scores[k, rx]]).astype(np.float64)
    return xs, ys, sc


def handcrafted_candidates(frame: np.ndarray, cfg):
    rows = strip_rows(frame.shape[0], cfg.strip_count, cfg.strip_weighting)
    sc = score_rows(frame, rows, cfg)
    return (*candidates_from_scores(sc, rows), rows, sc)


# ----------------------------------------------------------------------------
# learned scorer forward                      edgenet.py:67-83, 100-116, 182-233, 347-370
# ----------------------------------------------------------------------------
def rgbxy_windows(frame: np.ndarray, rows: list[int], mean, std) -> np.ndarray:
    """(S,5,7,W) float32 RGBXY windows; same values as make_rgbxy on the rows."""
    height, width = frame.shape[:2]
    r = np.asarray(rows, dtype=np.int64)
    win = r[:, None] + np.arange(-HALF, HALF + 1)[None, :]          # (S,7)
    rgb = frame[win].astype(np.float64)                              # (S,7,W,3)
    mean = np.asarray(mean, np.float64)
    std = np.asarray(std, np.float64)
    out = np.empty((len(rows), 5, 2 * HALF + 1, width), dtype=np.float32)
    out[:, :3] = ((rgb - mean) / std).transpose(0, 3, 1, 2)
    xs = (np.arange(width, dtype=np.float64) - (width - 1) / 2.0) / max(width - 1, 1)
    ys = (np.arange(height, dtype=np.float64) - (height - 1) / 2.0) / max(height - 1, 1)
    out[:, 3] = xs[None, None, :]
    out[:, 4] = ys[win][:, :, None]
    return out


def _valid_conv(x: np.ndarray, kern: np.ndarray, bias: np.ndarray) -> np.ndarray:
    """im2col cross-correlation in the reference's layout (edgenet.py:100-116)."""
    nb = x.shape[0]
    oc, _, kh, kw = kern.shape
    w = np.lib.stride_tricks.sliding_window_view(x, (kh, kw), axis=(2, 3))
    oh, ow = w.shape[2], w.shape[3]
    cols = np.ascontiguousarray(w.transpose(0, 2, 3, 1, 4, 5)).reshape(nb * oh * ow, -1)
    y = cols @ kern.reshape(oc, -1).T
    y += bias
    return y.reshape(nb, oh, ow, oc).transpose(0, 3, 1, 2)


def cnn_probs(windows: np.ndarray, layers) -> np.ndarray:
    """(S,W-6) float32 sigmoid probabilities; layers = [(kernel, bias)] * 4."""
    x = windows.astype(np.float32)
    for i, (kern, bias) in enumerate(layers):
        y = _valid_conv(x, kern.astype(np.float32), bias.astype(np.float32))
        x = y * (y > 0) if i < 3 else y
    z = x[:, 0, 0, :]
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    e = np.exp(z[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def learned_scores(frame: np.ndarray, rows, mean, std, layers) -> np.ndarray:
    width = frame.shape[1]
    probs = cnn_probs(rgbxy_windows(frame, rows, mean, std), layers)
    s = np.zeros((len(rows), width), dtype=np.float64)
    s[:, HALF:width - HALF] = probs
    return s


def glorot_layers(seed: int):
    """EdgeNet random init (edgenet.py:92-97, 149-159), float32."""
    rng = np.random.default_rng(seed)
    shapes = [(8, 5, 3, 3), (16, 8, 3, 3), (32, 16, 3, 3), (1, 32, 1, 1)]
    out = []
    for oc, ic, kh, kw in shapes:
        lim = np.sqrt(6.0 / (ic * kh * kw + oc * kh * kw))
        out.append((rng.uniform(-lim, lim, size=(oc, ic, kh, kw)).astype(np.float32),
                    np.zeros(oc, dtype=np.float32)))
    return out


# ----------------------------------------------------------------------------
# circle fitting                                             fitting.py:39-230
# ----------------------------------------------------------------------------
def keep_mask(xs, ys, scores, width, height, cfg) -> np.ndarray:
    """fitting.py:39-52: margin test on all four sides and the score floor."""
    xs = np.asarray(xs)
    ys = np.asarray(ys)
    edge = np.minimum(np.minimum(xs, width - 1 - xs), np.minimum(ys, height - 1 - ys))
    return (edge >= cfg.edge_margin_px) & (np.asarray(scores) >= cfg.min_point_score)


def sample_triplets(n: int, attempts: int, seed: int) -> np.ndarray:
    """fitting.py:147-156 (PCG64 keys, three smallest via argpartition)."""
    keys = np.random.default_rng(seed).random((attempts, n))
    return np.argpartition(keys, min(3, n - 1), axis=1)[:, :3]


def circumcircles(t: np.ndarray):
    """fitting.py:55-75 on (A,3,2) triplets."""
    ax, ay = t[:, 0, 0], t[:, 0, 1]
    ux0, uy0 = t[:, 1, 0] - ax, t[:, 1, 1] - ay
    vx0, vy0 = t[:, 2, 0] - ax, t[:, 2, 1] - ay
    det = ux0 * vy0 - uy0 * vx0
    scale = np.hypot(ux0, uy0) * np.hypot(vx0, vy0)
    good = (scale > 0) & (np.abs(det) > 1e-9 * scale)
    d = np.where(good, det, 1.0)
    hb = (ux0 * ux0 + uy0 * uy0) / 2.0
    hc = (vx0 * vx0 + vy0 * vy0) / 2.0
    ox = (hb * vy0 - hc * uy0) / d
    oy = (hc * ux0 - hb * vx0) / d
    rad = np.hypot(ox, oy)
    return ax + ox, ay + oy, rad, good & np.isfinite(rad) & (rad > 0)


def lsq_circles(p: np.ndarray, member: np.ndarray):
    """fitting.py:89-124: masked algebraic least squares via 3x3 normal eqs."""
    x, y = p[:, 0], p[:, 1]
    z = x * x + y * y
    mom = member.astype(np.float64) @ np.column_stack([x, y, z, x * x, x * y, y * y, x * z, y * z])
    sx, sy, sz, sxx, sxy, syy, sxz, syz = mom.T
    cnt = member.sum(axis=1).astype(np.float64)
    a = np.empty((len(mom), 3, 3))
    a[:, 0, 0], a[:, 1, 1], a[:, 2, 2] = 4.0 * sxx, 4.0 * syy, cnt
    a[:, 0, 1] = a[:, 1, 0] = 4.0 * sxy
    a[:, 0, 2] = a[:, 2, 0] = 2.0 * sx
    a[:, 1, 2] = a[:, 2, 1] = 2.0 * sy
    b = np.stack([2.0 * sxz, 2.0 * syz, sz], axis=1)
    det = (a[:, 0, 0] * (a[:, 1, 1] * a[:, 2, 2] - a[:, 1, 2] * a[:, 1, 2])
           - a[:, 0, 1] * (a[:, 0, 1] * a[:, 2, 2] - a[:, 1, 2] * a[:, 0, 2])
           + a[:, 0, 2] * (a[:, 0, 1] * a[:, 1, 2] - a[:, 1, 1] * a[:, 0, 2]))
    ok = (cnt >= 3) & np.isfinite(det) & (np.abs(det) > 1e-12 * np.maximum(cnt, 1.0) ** 3)
    a[~ok] = np.eye(3)
    sol = np.linalg.solve(a, b[..., None])[..., 0]
    r2 = sol[:, 2] + sol[:, 0] * sol[:, 0] + sol[:, 1] * sol[:, 1]
    ok &= np.isfinite(r2) & (r2 > 0)
    return sol[:, 0], sol[:, 1], np.sqrt(np.where(ok, r2, 1.0)), ok


def ransac(xs, ys, scores, width, height, cfg, seed=0, exhaustive=False, center=None):
    """fitting.py:159-230.  Returns (status, cx, cy, r, score, inliers)."""
    n = len(xs)
    if n < 3:
        return (NO_CANDIDATES, 0.0, 0.0, 0.0, 0.0, 0)
    pts = np.column_stack([np.asarray(xs, np.float64), np.asarray(ys, np.float64)])
    w8 = np.asarray(scores, dtype=np.float64)
    c0x, c0y = ((width - 1) / 2.0, (height - 1) / 2.0) if center is None else center
    p = (pts - (c0x, c0y)) / width
    tol = cfg.inlier_distance_px / width
    if exhaustive:
        tri = np.array(list(combinations(range(n), 3)), dtype=np.int64)
    else:
        tri = sample_triplets(n, cfg.ransac_attempts, seed)
    ccx, ccy, cr, live = circumcircles(p[tri])

    def inliers(live_now):
        d = np.abs(np.hypot(p[:, 0] - ccx[:, None], p[:, 1] - ccy[:, None]) - cr[:, None])
        return (d <= tol) & live_now[:, None]

    for _ in range(cfg.ransac_iterations):
        m = inliers(live)
        nx, ny, nr, ok = lsq_circles(p, m)
        live = live & ok
        ccx, ccy, cr = np.where(live, nx, ccx), np.where(live, ny, ccy), np.where(live, nr, cr)
    m = inliers(live)
    total = m.astype(np.float64) @ w8
    bad = (cr < cfg.min_radius_frac) | (cr > cfg.max_radius_frac) | (np.hypot(ccx, ccy) > cfg.max_center_offset_frac)
    ok = live & ~bad
    if not ok.any():
        return (GEOMETRY_GATE if (live & bad).any() else LOW_SCORE, 0.0, 0.0, 0.0, 0.0, 0)
    best = int(np.argmax(np.where(ok, total, -np.inf)))
    thr = cfg.min_circle_score if cfg.min_circle_score_absolute else cfg.min_circle_score * cfg.strip_count
    if total[best] < thr:
        return (LOW_SCORE, 0.0, 0.0, 0.0, 0.0, 0)
    return (ACCEPTED, float(c0x + ccx[best] * width), float(c0y + ccy[best] * width),
            float(cr[best] * width), float(total[best]), int(m[best].sum()))


# ----------------------------------------------------------------------------
# whole-frame estimate                                       estimator.py:55-74
# ----------------------------------------------------------------------------
def estimate(frame: np.ndarray, cfg, seed: int = 0, layers=None, norm=None):
    """(status, cx, cy, r, score, inliers) for one HWC uint8 frame."""
    height, width = frame.shape[:2]
    rows = strip_rows(height, cfg.strip_count, cfg.strip_weighting)
    if layers is None:
        sc = score_rows(frame, rows, cfg)
    else:
        sc = learned_scores(frame, rows, norm[0], norm[1], layers)
    xs, ys, s = candidates_from_scores(sc, rows)
    k = keep_mask(xs, ys, s, width, height, cfg)
    return ransac(xs[k], ys[k], s[k], width, height, cfg, seed)


# ----------------------------------------------------------------------------
# mask + crop                                    geometry.py:30-34, dataset.py:151-187
# ----------------------------------------------------------------------------
def disk_mask(cx: float, cy: float, r: float, height: int, width: int) -> np.ndarray:
    """uint8 (H,W): 1 where dx*dx + dy*dy <= r*r at integer pixel centres."""
    dx = np.arange(width, dtype=np.float64)[None, :] - cx
    dy = np.arange(height, dtype=np.float64)[:, None] - cy
    return ((dx * dx + dy * dy) <= r * r).astype(np.uint8)


def crop_bounds(cx: float, cy: float, r: float, width: int, height: int):
    """Inclusive (x0, y0, x1, y1) of crop_augment's rectangle, or None."""
    def inside(x, y):
        dx, dy = x - cx, y - cy
        return dx * dx + dy * dy <= r * r

    if all(inside(x, y) for x, y in ((0, 0), (width - 1, 0), (0, height - 1), (width - 1, height - 1))):
        return None
    half = r / math.sqrt(2.0)
    capx, capy = min(cx, width - 1 - cx), min(cy, height - 1 - cy)
    wx, wy = min(half, capx), min(half, capy)
    if wx < half:
        wy = min(capy, math.sqrt(max(r ** 2 - wx * wx, 0.0)))
    elif wy < half:
        wx = min(capx, math.sqrt(max(r ** 2 - wy * wy, 0.0)))
    x0, x1 = max(math.ceil(cx - wx), 0), min(math.floor(cx + wx), width - 1)
    y0, y1 = max(math.ceil(cy - wy), 0), min(math.floor(cy + wy), height - 1)
    if x1 - x0 + 1 < MIN_CROP or y1 - y0 + 1 < MIN_CROP:
        return None
    return (x0, y0, x1, y1)


# ----------------------------------------------------------------------------
# normalised-Hausdorff evaluation                            metrics.py:52-223
# ----------------------------------------------------------------------------
REF_DIAGONAL = math.hypot(1920.0, 1080.0)   # metrics.py:23


def _linspace_cols(x0: float, dx: float, y0: float, dy: float, n: int) -> np.ndarray:
    ts = np.linspace(0.0, 1.0, n + 1)
    return np.column_stack((x0 + ts * dx, y0 + ts * dy))


def boundary_pieces(circle, width: int, height: int):
    """Arcs (t0, t1) then covered edge runs ((x0, y0), (x1, y1)) of the border of
    disk ∩ [0, W-1] x [0, H-1] (metrics.py:52-130).  circle = (cx, cy, r) or None."""
    xhi, yhi = float(width - 1), float(height - 1)
    if circle is None:
        return [], [((0.0, 0.0), (xhi, 0.0)), ((xhi, 0.0), (xhi, yhi)),
                     ((xhi, yhi), (0.0, yhi)), ((0.0, yhi), (0.0, 0.0))]
    cx, cy, r = circle
    tau = 2.0 * math.pi
    cross = []
    for b in (0.0, xhi):                                  # metrics.py:58-62
        c = (b - cx) / r
        if -1.0 <= c <= 1.0:
            t = math.acos(c)
            cross += [t, tau - t]
    for b in (0.0, yhi):                                  # metrics.py:63-67
        s = (b - cy) / r
        if -1.0 <= s <= 1.0:
            t = math.asin(s)
            cross += [t % tau, (math.pi - t) % tau]

    def inside(t):
        x, y = cx + r * math.cos(t), cy + r * math.sin(t)
        return 0.0 <= x <= xhi and 0.0 <= y <= yhi

    arcs = []
    if not cross:
        if inside(0.0):
            arcs = [(0.0, tau)]
    else:
        ts = sorted(set(cross))
        for k, t0 in enumerate(ts):
            t1 = ts[k + 1] if k + 1 < len(ts) else ts[0] + tau
            if t1 - t0 > 1e-12 and inside((t0 + t1) / 2.0):
                arcs.append((t0, t1))
    runs = []
    for fixed, hi, horiz in ((0.0, xhi, True), (yhi, xhi, True), (0.0, yhi, False), (xhi, yhi, False)):
        rad2 = r * r - ((fixed - cy) ** 2 if horiz else (fixed - cx) ** 2)   # metrics.py:104
        if rad2 < 0.0:
            continue
        half = math.sqrt(rad2)
        mid = cx if horiz else cy
        a, b = max(0.0, mid - half), min(hi, mid + half)
        if b <= a:
            continue
        runs.append(((a, fixed), (b, fixed)) if horiz else ((fixed, a), (fixed, b)))
    return arcs, runs


def boundary_points(circle, width: int, height: int, spacing: float = 1.0) -> np.ndarray:
    """metrics.py:148-176 (samples: _sample_segment :133-138, _sample_arc :141-146)."""
    arcs, runs = boundary_pieces(circle, width, height)
    chunks = []
    for t0, t1 in arcs:
        cx, cy, r = circle
        n = max(1, math.ceil(r * (t1 - t0) / spacing))
        ts = np.linspace(t0, t1, n + 1)
        chunks.append(np.column_stack((cx + r * np.cos(ts), cy + r * np.sin(ts))))
    for p0, p1 in runs:
        n = max(1, math.ceil(math.hypot(p1[0] - p0[0], p1[1] - p0[1]) / spacing))
        chunks.append(_linspace_cols(p0[0], p1[0] - p0[0], p0[1], p1[1] - p0[1], n))
    if not chunks:
        return np.zeros((0, 2))
    return np.vstack(chunks)


def hausdorff(a: np.ndarray, b: np.ndarray, block: int = 2048) -> float:
    """Symmetric Hausdorff distance (metrics.py:193-203) by brute force:
    sqrt(dx*dx + dy*dy), the p=2 distance the reference's KD-tree returns."""
    def directed(p, q):
        best = 0.0
        for i in range(0, len(p), block):
            dx = p[i:i + block, None, 0] - q[None, :, 0]
            dy = p[i:i + block, None, 1] - q[None, :, 1]
            best = max(best, float(np.sqrt((dx * dx + dy * dy).min(axis=1)).max()))
        return best
    return max(directed(a, b), directed(b, a))


def area_error_px(pred, truth, width: int, height: int, spacing: float = 1.0) -> float:
    """metrics.py:206-223; pred / truth = (cx, cy, r) or None (full frame)."""
    hd = hausdorff(boundary_points(pred, width, height, spacing),
                   boundary_points(truth, width, height, spacing))
    return REF_DIAGONAL / math.hypot(width, height) * hd


def hausdorff_kdtree(a: np.ndarray, b: np.ndarray) -> float:
    """metrics.py:193-203 verbatim in algorithm (scipy cKDTree both ways): the
    CPU baseline's timed form of ``hausdorff``; same values."""
    from scipy.spatial import cKDTree
    return float(max(cKDTree(b).query(a)[0].max(), cKDTree(a).query(b)[0].max()))


def area_error_px_kdtree(pred, truth, width: int, height: int) -> float:
    hd = hausdorff_kdtree(boundary_points(pred, width, height), boundary_points(truth, width, height))
    return REF_DIAGONAL / math.hypot(width, height) * hd


# ----------------------------------------------------------------------------
# learned-variant training                     edgenet.py:100-130, 182-225, 236-344
# ----------------------------------------------------------------------------
def _im2col(x: np.ndarray, kh: int, kw: int) -> np.ndarray:
    w = np.lib.stride_tricks.sliding_window_view(x, (kh, kw), axis=(2, 3))
    return np.ascontiguousarray(w.transpose(0, 2, 3, 1, 4, 5)).reshape(-1, x.shape[1] * kh * kw)


def forward_logits(x: np.ndarray, layers):
    """(B,5,h,W) -> logits (B,1,h-6,W-6) and the per-layer caches
    (input, im2col, ReLU mask) of edgenet.py:182-205."""
    x = np.asarray(x, dtype=np.float32)
    caches = []
    for i, (kern, bias) in enumerate(layers):
        y = _valid_conv(x, kern, bias)
        mask = (y > 0) if i < 3 else None
        caches.append((x.shape, _im2col(x, kern.shape[2], kern.shape[3]), mask))
        x = y * mask if i < 3 else y
    return x, caches


def backward(dlogits: np.ndarray, caches, layers):
    """Per-layer (dkernel, dbias), edgenet.py:119-130 + 213-224."""
    grads = [None] * 4
    dy = dlogits.astype(np.float32)
    for k in range(3, -1, -1):
        x_shape, cols, _ = caches[k]
        kern = layers[k][0]
        oc, ic, kh, kw = kern.shape
        dy_mat = np.ascontiguousarray(dy.transpose(0, 2, 3, 1)).reshape(-1, oc)
        grads[k] = ((dy_mat.T @ cols).reshape(kern.shape), dy_mat.sum(axis=0))
        padded = np.pad(dy, ((0, 0), (0, 0), (kh - 1, kh - 1), (kw - 1, kw - 1)))
        flipped = np.ascontiguousarray(kern[:, :, ::-1, ::-1].transpose(1, 0, 2, 3))
        dy = _valid_conv(padded, flipped, np.zeros(ic, dtype=np.float32))
        if k > 0:
            dy = dy * caches[k - 1][2]
    return grads


def sigmoid32(z: np.ndarray) -> np.ndarray:
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    e = np.exp(z[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def bce_with_logits(logits: np.ndarray, targets: np.ndarray) -> float:
    """edgenet.py:236-241: mean stable BCE in float64."""
    z = logits.astype(np.float64)
    t = targets.astype(np.float64)
    return float((np.maximum(z, 0.0) - z * t + np.log1p(np.exp(-np.abs(z)))).mean())


def train_step(x, t, layers, lr: float):
    """One SGD step of edgenet.train (:306-328); returns (loss, grads, new layers)."""
    logits, caches = forward_logits(x, layers)
    loss = bce_with_logits(logits, t)
    dlog = (sigmoid32(logits) - t.astype(np.float32)) / logits.size
    grads = backward(dlog, caches, layers)
    new = [(k - np.float32(lr) * dk, b - np.float32(lr) * db) for (k, b), (dk, db) in zip(layers, grads)]
    return loss, grads, new


def train(layers, train_x, train_t, val_x, val_t, lr=0.001, batch=8, patience=5, epochs=50,
          shuffle=True, seed=0):
    """edgenet.train (:277-344): SGD, per-epoch permutation, early stopping on
    the validation loss; returns (layers of the best epoch, train losses, val
    losses, best epoch).  Raises FloatingPointError on a non-finite loss."""
    rng = np.random.default_rng(seed)
    layers = [(k.copy(), b.copy()) for k, b in layers]
    best, best_val, stale, best_epoch = [(k.copy(), b.copy()) for k, b in layers], np.inf, 0, -1
    tl, vl = [], []
    for epoch in range(epochs):
        order = rng.permutation(len(train_x)) if shuffle else np.arange(len(train_x))
        tot, cnt = 0.0, 0
        for s in range(0, len(order), batch):
            idx = order[s:s + batch]
            x, t = train_x[idx], train_t[idx]
            logits, caches = forward_logits(x, layers)
            loss = bce_with_logits(logits, t)
            if not np.isfinite(loss):
                raise FloatingPointError(f"non-finite loss at epoch {epoch}, sample offset {s}")
            tot += loss * logits.size
            cnt += logits.size
            dlog = (sigmoid32(logits) - t.astype(np.float32)) / logits.size
            grads = backward(dlog, caches, layers)
            if lr != 0.0:
                for (k, b), (dk, db) in zip(layers, grads):
                    k -= lr * dk
                    b -= lr * db
        tl.append(tot / cnt)
        if val_x is not None:
            vt, vc = 0.0, 0
            vb = max(batch, 32)
            for s in range(0, len(val_x), vb):
                lg, _ = forward_logits(val_x[s:s + vb], layers)
                vt += bce_with_logits(lg, val_t[s:s + vb]) * lg.size
                vc += lg.size
            v = vt / max(vc, 1)
            vl.append(v)
            if v < best_val:
                best_val, best, best_epoch, stale = v, [(k.copy(), b.copy()) for k, b in layers], epoch, 0
            else:
                stale += 1
                if stale >= patience:
                    break
        else:
            best, best_epoch = [(k.copy(), b.copy()) for k, b in layers], epoch
    return best, tl, vl, best_epoch
