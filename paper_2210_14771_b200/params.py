"""Pipeline tunables with the paper's defaults.

Same field names, defaults and validation as the reference's ``EcaConfig``
(/root/reference/pkg/src/eca/config.py:14-78).  :meth:`EcaConfig.device_params`
packs it into the POD ``EcaParams`` struct of ``include/eca_b200.h`` that every
kernel receives by value.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

_POSITIVE = ("gradient_threshold", "angle_threshold_deg", "intensity_threshold",
             "min_point_score", "inlier_distance_px", "min_circle_score",
             "min_radius_frac", "max_radius_frac", "max_center_offset_frac")


@dataclass(frozen=True, slots=True)
class EcaConfig:
    strip_count: int = 16
    strip_weighting: float = 8.0
    gradient_threshold: float = 20.0
    angle_threshold_deg: float = 30.0
    intensity_threshold: float = 25.0
    edge_margin_px: int = 3
    min_point_score: float = 0.03
    inlier_distance_px: float = 3.0
    min_circle_score: float = 0.06
    min_circle_score_absolute: bool = False
    min_radius_frac: float = 0.1
    max_radius_frac: float = 0.8
    max_center_offset_frac: float = 0.2
    ransac_attempts: int = 32
    ransac_iterations: int = 3

    def __post_init__(self) -> None:   # config.py:41-66
        if self.strip_count < 4:
            raise ValueError(f"strip_count must be >= 4, got {self.strip_count}")
        if self.strip_weighting <= 0:
            raise ValueError(f"strip_weighting must be positive, got {self.strip_weighting}")
        for name in _POSITIVE:
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive, got {getattr(self, name)}")
        if self.edge_margin_px < 0:
            raise ValueError(f"edge_margin_px must be >= 0, got {self.edge_margin_px}")
        if self.min_radius_frac >= self.max_radius_frac:
            raise ValueError(f"min_radius_frac must be < max_radius_frac, got "
                             f"{self.min_radius_frac} >= {self.max_radius_frac}")
        if self.ransac_attempts < 1 or self.ransac_iterations < 1:
            raise ValueError("ransac_attempts and ransac_iterations must be >= 1")

    def circle_score_threshold(self) -> float:
        """Absolute inlier-score sum a fit needs (config.py:69-73)."""
        if self.min_circle_score_absolute:
            return self.min_circle_score
        return self.min_circle_score * self.strip_count

    def device_params(self, width: int, height: int, center=None) -> "EcaParams":
        """POD copy for the kernels; derived constants use the reference's
        evaluation order so the GPU sees the same doubles numpy does."""
        ang = 180.0 / (math.pi * self.angle_threshold_deg)          # handcrafted.py:178
        cx, cy = ((width - 1) / 2.0, (height - 1) / 2.0) if center is None else center
        return EcaParams(
            width=width, height=height, strip_count=self.strip_count,
            edge_margin_px=self.edge_margin_px, ransac_attempts=self.ransac_attempts,
            ransac_iterations=self.ransac_iterations,
            gradient_threshold=self.gradient_threshold,
            intensity_threshold=self.intensity_threshold,
            angle_scale=ang, zero_grad_angle=math.pi * ang,
            min_point_score=self.min_point_score,
            inlier_tol=self.inlier_distance_px / width,
            circle_score_threshold=self.circle_score_threshold(),
            min_radius_frac=self.min_radius_frac, max_radius_frac=self.max_radius_frac,
            max_center_offset_frac=self.max_center_offset_frac,
            center_x=cx, center_y=cy,
        )


class EcaParams(ctypes.Structure):
    """ctypes mirror of ``struct EcaParams`` (include/eca_b200.h)."""

    _fields_ = [
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("strip_count", ctypes.c_int32), ("edge_margin_px", ctypes.c_int32),
        ("ransac_attempts", ctypes.c_int32), ("ransac_iterations", ctypes.c_int32),
        ("gradient_threshold", ctypes.c_double), ("intensity_threshold", ctypes.c_double),
        ("angle_scale", ctypes.c_double), ("zero_grad_angle", ctypes.c_double),
        ("min_point_score", ctypes.c_double), ("inlier_tol", ctypes.c_double),
        ("circle_score_threshold", ctypes.c_double),
        ("min_radius_frac", ctypes.c_double), ("max_radius_frac", ctypes.c_double),
        ("max_center_offset_frac", ctypes.c_double),
        ("center_x", ctypes.c_double), ("center_y", ctypes.c_double),
    ]


_DEFAULT: EcaConfig | None = None


def config_default() -> EcaConfig:
    """The default configuration (config.py:76-77).  EcaConfig is frozen, so
    one shared instance is returned (built once: construction validates)."""
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = EcaConfig()
    return _DEFAULT
