"""B200-native endoscopic content-area estimation (arXiv 2210.14771).

Drop-in for the reference package ``eca`` (/root/reference/pkg/src/eca/__init__.py:10-65)
on the hot path: strip edge scoring (handcrafted and learned), candidate
filtering, seeded RANSAC circle fitting, masks and crops, all as sm_100a CUDA
kernels in ``libeca_b200.so`` behind a C ABI (include/eca_b200.h).
"""

from .api import (
    HANDCRAFTED,
    Accepted,
    EstimatorVariant,
    FitResult,
    FrameError,
    Handcrafted,
    Learned,
    Rejected,
    RejectionReason,
    StripScoreRow,
    crop_area,
    crop_augment,
    crop_bounds,
    draw_mask,
    estimate,
    estimate_area,
    estimate_batch,
    filter_candidates,
    fit_area,
    get_points,
    get_points_batch,
    ransac_fit,
    records_to_fits,
    score_frame_strips,
    strip_heights,
    triplet_table,
    validate_frame,
)
from .engine import ContentAreaEngine
from .params import EcaConfig, config_default
from .shapes import (
    FULL_FRAME,
    Circle,
    CircularArea,
    ContentArea,
    EdgeCandidate,
    FullFrame,
    Side,
    circle_contains,
    frame_center,
)
from .stripnet import (
    ChannelStats,
    CorruptWeightsError,
    EdgeNet,
    compute_channel_stats,
    load_weights,
    load_weights_file,
    save_weights,
    save_weights_file,
)

from . import labels, metrics, training
from .labels import EcaAnnotation, Source, pseudo_label
from .metrics import area_error_px, area_errors, evaluate_dataset

__version__ = "0.1.0"
