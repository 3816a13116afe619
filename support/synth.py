"""Deterministic synthetic endoscopic frames (input generator for tests and bench).

Restates the reference renderer ``eca.dataset.render_synthetic`` /
``benchmark_spec(s)`` (/root/reference/pkg/src/eca/dataset.py:228-444) so the
GPU box can produce the BASELINE.json workloads without the reference tree.
All randomness is integer draws from numpy's PCG64, so a frame is identical
bytes to the reference's render of the same spec and seed; the SHA-256 pin of
``tests/golden`` checks that.  Not on the hot path: frames are produced once,
before any timing.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2210_14771_b200.shapes import Circle

CATEGORIES = ("clean", "dark", "bleed", "overlay", "corner")     # dataset.py:359


@dataclass(frozen=True, slots=True)
class BleedSpot:
    """Saturated glow on the content edge (dataset.py:228-235)."""

    angle_deg: float
    radius_px: float
    brightness: int


@dataclass(frozen=True, slots=True)
class BoxOverlay:
    """Flat burned-in rectangle, inclusive bounds (dataset.py:238-246)."""

    x0: int
    y0: int
    x1: int
    y1: int
    brightness: int


@dataclass(frozen=True, slots=True)
class SyntheticSpec:
    """Frame recipe (dataset.py:248-275), including the geometry-gate check."""

    width: int = 960
    height: int = 540
    circle: Circle | None = None
    border_noise_sigma: float = 2.0
    content_brightness: int = 150
    texture_amplitude: int = 40
    bleed: BleedSpot | None = None
    overlay: BoxOverlay | None = None
    adversarial: bool = False

    def __post_init__(self) -> None:
        c = self.circle
        if c is None or self.adversarial:
            return
        off = math.hypot(c.cx - (self.width - 1) / 2.0, c.cy - (self.height - 1) / 2.0)
        # default gates: r in [0.1, 0.8] * W, centre offset <= 0.2 * W
        if not (0.1 * self.width <= c.r <= 0.8 * self.width) or off > 0.2 * self.width:
            raise ValueError(f"{c} violates the geometry gates; set adversarial=True to keep it")


def _lattice_noise(rng, h: int, w: int, cell: int, amp: int) -> np.ndarray:
    """Integer bilinear value noise (dataset.py:278-297)."""
    if amp <= 0:
        return np.zeros((h, w), dtype=np.int64)
    grid = rng.integers(-amp, amp + 1, size=(h // cell + 2, w // cell + 2), dtype=np.int64)
    yi, yf = np.divmod(np.arange(h), cell)
    xi, xf = np.divmod(np.arange(w), cell)
    wy0 = (cell - yf)[:, None]
    wy1 = yf[:, None]
    left = grid[np.ix_(yi, xi)] * wy0 + grid[np.ix_(yi + 1, xi)] * wy1
    right = grid[np.ix_(yi, xi + 1)] * wy0 + grid[np.ix_(yi + 1, xi + 1)] * wy1
    return (left * (cell - xf)[None, :] + right * xf[None, :]) // (cell * cell)


def _border_noise(rng, shape, sigma: float) -> np.ndarray:
    """Sum of four uniform integer draws minus its mean (dataset.py:300-307)."""
    if sigma <= 0:
        return np.zeros(shape, dtype=np.int64)
    m = max(1, round(math.sqrt(1.0 + 3.0 * sigma * sigma) - 1.0))
    return rng.integers(0, m + 1, size=(4, *shape), dtype=np.int64).sum(axis=0) - 2 * m


def render(spec: SyntheticSpec, rng_seed: int) -> np.ndarray:
    """(H, W, 3) uint8 frame for ``spec`` (dataset.py:310-356)."""
    rng = np.random.default_rng(rng_seed)
    h, w = spec.height, spec.width
    g = spec.content_brightness + _lattice_noise(rng, h, w, 24, spec.texture_amplitude)
    np.clip(g, 0, 255, out=g)
    c = spec.circle
    if c is not None:
        ddx = np.arange(w, dtype=np.float64)[None, :] - c.cx
        ddy = np.arange(h, dtype=np.float64)[:, None] - c.cy
        d2 = ddx * ddx + ddy * ddy
        rim = np.clip(_border_noise(rng, (h, w), spec.border_noise_sigma), 0, 255)
        g = np.where(d2 <= c.r * c.r, g, rim)
        b = spec.bleed
        if b is not None:
            phi = math.radians(b.angle_deg)
            px, py = c.cx + c.r * math.cos(phi), c.cy + c.r * math.sin(phi)
            glow = (np.arange(w, dtype=np.float64)[None, :] - px) ** 2 + (
                np.arange(h, dtype=np.float64)[:, None] - py) ** 2
            g = np.where((d2 > c.r * c.r) & (glow <= b.radius_px ** 2), b.brightness, g)
    o = spec.overlay
    if o is not None:
        g[max(o.y0, 0):o.y1 + 1, max(o.x0, 0):o.x1 + 1] = o.brightness
    out = np.empty((h, w, 3), dtype=np.uint8)
    out[..., 0] = g
    out[..., 1] = g * 205 // 256
    out[..., 2] = g * 178 // 256
    return out


def bench_spec(category: str, rng, width: int = 960, height: int = 540) -> SyntheticSpec:
    """One randomised spec of a benchmark category (dataset.py:362-432)."""
    cx0, cy0 = (width - 1) / 2.0, (height - 1) / 2.0

    def disk(r_lo, r_hi, off_hi):
        r = rng.uniform(r_lo, r_hi) * width
        a = rng.uniform(0.0, 2.0 * math.pi)
        off = rng.uniform(0.0, off_hi) * width
        return Circle(cx0 + off * math.cos(a), cy0 + off * math.sin(a), r)

    if category == "clean":
        return SyntheticSpec(width, height, circle=disk(0.30, 0.45, 0.07),
                             border_noise_sigma=rng.uniform(0.0, 3.0),
                             content_brightness=int(rng.integers(120, 200)))
    if category == "dark":
        return SyntheticSpec(width, height, circle=disk(0.30, 0.45, 0.07),
                             border_noise_sigma=rng.uniform(0.0, 2.0),
                             content_brightness=int(rng.integers(36, 60)), texture_amplitude=12)
    if category == "bleed":
        c = disk(0.30, 0.42, 0.06)
        sigma = rng.uniform(0.0, 2.0)
        bright = int(rng.integers(120, 200))
        spot = BleedSpot(rng.uniform(0.0, 360.0), rng.uniform(12.0, 30.0), int(rng.integers(120, 230)))
        return SyntheticSpec(width, height, circle=c, border_noise_sigma=sigma,
                             content_brightness=bright, bleed=spot)
    if category == "overlay":
        bw, bh = int(0.22 * width), int(0.12 * height)
        corner = rng.integers(0, 4)
        x0 = 0 if corner % 2 == 0 else width - bw
        y0 = 0 if corner < 2 else height - bh
        c = disk(0.32, 0.45, 0.06)
        sigma = rng.uniform(0.0, 2.0)
        bright = int(rng.integers(120, 200))
        box = BoxOverlay(x0, y0, x0 + bw - 1, y0 + bh - 1, int(rng.integers(60, 110)))
        return SyntheticSpec(width, height, circle=c, border_noise_sigma=sigma,
                             content_brightness=bright, overlay=box)
    if category == "corner":
        off = rng.uniform(0.11, 0.18) * width
        sign = 1.0 if rng.integers(0, 2) else -1.0
        near = math.hypot(width / 2.0 - off, height / 2.0)
        far = math.hypot(width / 2.0 + off, height / 2.0)
        r = rng.uniform(near * 1.03, min(far * 0.97, 0.78 * width))
        return SyntheticSpec(width, height, circle=Circle(cx0 + sign * off, cy0, r),
                             border_noise_sigma=rng.uniform(0.0, 2.0),
                             content_brightness=int(rng.integers(110, 190)))
    raise ValueError(f"unknown benchmark category {category!r}")


def bench_specs(count: int, width: int = 960, height: int = 540, seed: int = 0):
    """``count`` (category, spec) pairs cycling CATEGORIES (dataset.py:435-444)."""
    rng = np.random.default_rng(seed)
    return [(CATEGORIES[k % 5], bench_spec(CATEGORIES[k % 5], rng, width, height))
            for k in range(count)]


# ---------------------------------------------------------------------------
# BASELINE.json workloads
# ---------------------------------------------------------------------------
def c1_frame(width: int = 1920, height: int = 1080) -> np.ndarray:
    """The reference's ``eca bench`` frame (cli.py:381-383)."""
    return render(bench_spec("clean", np.random.default_rng(0), width, height), 0)


def c2_frame(k: int, width: int = 1920, height: int = 1080, seed: int = 2024, specs=None) -> np.ndarray:
    """Frame k of the batched mix: spec k of bench_specs(.., seed), rng_seed 30000+k."""
    specs = specs or bench_specs(k + 1, width, height, seed)
    return render(specs[k][1], 30000 + k)


def c4_frames(width: int = 3840, height: int = 2160) -> dict[str, np.ndarray]:
    """4K edge cases: full circle, rectangle, heavy noise +
    box overlay + OSD text, no content.  Pinned by tests/golden (c4_* cases)."""
    cx0, cy0 = (width - 1) / 2.0, (height - 1) / 2.0
    noisy = render(SyntheticSpec(width, height, circle=Circle(cx0 + 100, cy0 - 50, 0.38 * width),
                                 border_noise_sigma=12, overlay=BoxOverlay(0, 0, 843, 258, 90)), 7)
    return {
        "full_circle": render(SyntheticSpec(width, height, circle=Circle(cx0, cy0, 0.26 * width)), 7),
        "rectangle": render(SyntheticSpec(width, height, circle=None), 7),
        "heavy_noise": noisy,
        "heavy_noise_text": stamp_osd_text(noisy, seed=7),
        "all_zeros": np.zeros((height, width, 3), dtype=np.uint8),
        "uniform_128": np.full((height, width, 3), 128, dtype=np.uint8),
        "dark_noise": np.random.default_rng(3).integers(0, 12, (height, width, 3)).astype(np.uint8),
    }


def stamp_osd_text(frame: np.ndarray, seed: int) -> np.ndarray:
    """Burn deterministic on-screen-display "text" into a copy of the frame:
    four lines of 24 random 5x7 block glyphs (one blank column between
    glyphs), scaled by max(2, W // 640), two lines at the top left and two at
    the bottom right, brightness 235 / 215 / 195 / 175.  Integer-only, so the
    golden generator (tests/golden/make_golden_configs.py) and the tests build
    identical bytes; the text crosses strip rows on both sides."""
    rng = np.random.default_rng(seed)
    f = frame.copy()
    h, w = f.shape[:2]
    cell = max(2, w // 640)
    for line, (x0, y0) in enumerate([(40, 300), (40, 360), (w - 900, h - 200), (w - 900, h - 140)]):
        bits = rng.integers(0, 2, size=(7, 6 * 24)).astype(bool)
        bits[:, 5::6] = False                       # inter-glyph gap
        ys, xs = np.nonzero(np.kron(bits, np.ones((cell, cell), dtype=bool)))
        ys, xs = ys + y0, xs + x0
        ok = (ys >= 0) & (xs >= 0) & (ys < h) & (xs < w)
        f[ys[ok], xs[ok]] = 235 - 20 * line
    return f
