"""GPU parity of the evaluation row (metrics.py:148-283) against
the reference's golden fixtures (tests/golden/make_golden_metrics.py) and the
CPU oracle.

Tolerances: boundary sample counts exact; sample coordinates within 1e-9 px
(CUDA cos/sin/acos/asin vs the host libm differ by an ulp or two); Hausdorff
distances of the same point sets bit-exact (sqrt(dx*dx + dy*dy) in FP64, the
KD-tree's p=2 distance); distances between boundaries within 1e-9 px; miss
classes and report percentages exact.
"""

import math

import numpy as np
import pytest
import torch

import paper_2210_14771_b200 as eb
from oracle import eca_oracle as orc
from paper_2210_14771_b200 import metrics as gm

from ._fixtures import load_json, load_npz

pytestmark = pytest.mark.gpu
PT_TOL = 1e-9


def _area(c):
    return eb.FULL_FRAME if c is None else eb.Circle(*c)


def test_boundary_points_match_reference():
    g, pts = load_json("metrics.json"), load_npz("metrics_points.npz")
    for i, c in enumerate(g["cases"]):
        for side, key in (("pred", "p"), ("truth", "t")):
            got = gm.boundary_points(_area(c[side]), c["w"], c["h"], c["spacing"])
            assert len(got) == c[f"n_{side}"], (i, side, c)
            want = pts[f"{key}{i}"] if f"{key}{i}" in pts else \
                orc.boundary_points(None if c[side] is None else tuple(c[side]), c["w"], c["h"], c["spacing"])
            assert np.abs(got - want).max() <= PT_TOL, (i, side, np.abs(got - want).max())


def test_boundary_length_matches_reference():
    for c in load_json("metrics.json")["cases"]:
        assert gm.boundary_length(_area(c["pred"]), c["w"], c["h"]) == pytest.approx(c["len_pred"], rel=1e-12)
        assert gm.boundary_length(_area(c["truth"]), c["w"], c["h"]) == pytest.approx(c["len_truth"], rel=1e-12)


def test_hausdorff_point_sets_bit_exact():
    g, pts = load_json("metrics.json"), load_npz("metrics_points.npz")
    for k, s in enumerate(g["sets"]):
        assert gm.hausdorff(pts[f"ha{k}"], pts[f"hb{k}"]) == s["hd"], k
    # the reference's own unit cases (test_metrics.py:92-104)
    a = np.random.default_rng(0).uniform(0, 100, (50, 2))
    assert gm.hausdorff(a, a) == 0.0
    assert gm.hausdorff(np.array([[0.0, 0.0]]), np.array([[3.0, 4.0]])) == 5.0
    with pytest.raises(ValueError):
        gm.hausdorff(np.empty((0, 2)), np.array([[0.0, 0.0]]))


def test_hausdorff_random_sets_match_oracle():
    rng = np.random.default_rng(11)
    for k in range(30):
        a = rng.uniform(-1e3, 1e3, (int(rng.integers(1, 3000)), 2))
        b = a[: max(1, len(a) // 2)] + rng.normal(0, 0.5, (max(1, len(a) // 2), 2)) if k % 3 == 0 else \
            rng.uniform(-1e3, 1e3, (int(rng.integers(1, 3000)), 2))
        assert gm.hausdorff(a, b) == orc.hausdorff(a, b), k


def test_area_errors_match_reference():
    g = load_json("metrics.json")
    cs = g["cases"]
    for sp in sorted({c["spacing"] for c in cs}):
        sel = [c for c in cs if c["spacing"] == sp]
        for w, h in sorted({(c["w"], c["h"]) for c in sel}):
            grp = [c for c in sel if (c["w"], c["h"]) == (w, h)]
            nh = gm.area_errors([_area(c["pred"]) for c in grp], [_area(c["truth"]) for c in grp], (w, h),
                                spacing=sp)
            for c, v in zip(grp, nh):
                assert abs(v - c["nh"]) <= PT_TOL * 10, (c, v)
    # mixed frame sizes in one batch
    nh = gm.area_errors([_area(c["pred"]) for c in cs if c["spacing"] == 1.0],
                        [_area(c["truth"]) for c in cs if c["spacing"] == 1.0],
                        [(c["w"], c["h"]) for c in cs if c["spacing"] == 1.0])
    want = [c["nh"] for c in cs if c["spacing"] == 1.0]
    assert np.abs(nh - np.array(want)).max() <= 1e-8


def test_area_error_px_single_and_errors():
    c = load_json("metrics.json")["cases"][1]
    assert gm.area_error_px(_area(c["pred"]), _area(c["truth"]), c["w"], c["h"]) == \
        pytest.approx(c["nh"], abs=1e-8)
    with pytest.raises(ValueError, match="does not intersect"):
        gm.area_error_px(eb.Circle(-500.0, -500.0, 10.0), eb.FULL_FRAME, 100, 100)
    with pytest.raises(ValueError, match="does not intersect"):
        gm.boundary_points(eb.Circle(-500.0, -500.0, 10.0), 100, 100)
    with pytest.raises(ValueError, match="degenerate"):
        gm.boundary_points(eb.FULL_FRAME, 1, 100)


def test_evaluate_dataset_matches_reference():
    r = load_json("metrics.json")["report"]
    preds = {i: _area(p) for i, p in zip(r["ids"], r["pred"])}
    truths = {i: _area(t) for i, t in zip(r["ids"], r["truth"])}
    rep = gm.evaluate_dataset(preds, truths, (1920, 1080))
    assert [s.label.value for s in rep.per_sample] == r["labels"]
    assert rep.avg_error_px == pytest.approx(r["avg"], abs=1e-9)
    assert (rep.miss_pct, rep.bad_miss_pct) == (r["miss"], r["bad"])
    assert gm.report_markdown({"handcrafted": rep}) == r["markdown"]
    with pytest.raises(ValueError, match="unmatched"):
        gm.evaluate_dataset({"a": None}, {"b": None}, (100, 100))


def test_evaluate_dataset_reference_unit_cases():
    # test_metrics.py:183-213
    truth = {k: eb.Circle(960.0, 540.0, 300.0) for k in "abcd"}
    preds = dict(truth)
    preds["c"] = eb.Circle(960.0, 540.0, 320.0)
    preds["d"] = eb.Circle(960.0, 540.0, 330.0)
    rep = gm.evaluate_dataset(preds, truth, (1920, 1080))
    assert rep.miss_pct == pytest.approx(50.0) and rep.bad_miss_pct == pytest.approx(25.0)
    perfect = gm.evaluate_dataset({"a": eb.Circle(960.0, 540.0, 400.0), "b": None},
                                  {"a": eb.Circle(960.0, 540.0, 400.0), "b": None}, (1920, 1080))
    assert perfect.avg_error_px == 0.0


def test_fitted_records_evaluate_against_truth():
    """The evaluation consumes the hot path's records directly (estimate ->
    area_errors), as the paper's accuracy tables do."""
    from support import synth
    specs = synth.bench_specs(8, 640, 480, seed=2024)
    frames = np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])
    areas = eb.estimate_batch(list(frames))
    truth = [s.circle for _, s in specs]
    nh = gm.area_errors(areas, truth, (640, 480))
    for a, t, v in zip(areas, truth, nh):
        want = orc.area_error_px(None if not isinstance(a, eb.CircularArea) else
                                 (a.circle.cx, a.circle.cy, a.circle.r),
                                 None if t is None else (t.cx, t.cy, t.r), 640, 480)
        assert abs(v - want) <= 1e-8, (a, t, v, want)


try:
    from hypothesis import given, settings
    from hypothesis import strategies as st
except ImportError:   # pragma: no cover
    given = None

if given is not None:
    @given(data=st.data())
    @settings(max_examples=40, deadline=None)
    def test_hausdorff_metric_axioms(data):
        """test_metrics.py:113-131 on the GPU distance: symmetry, identity,
        triangle inequality, and equality with the oracle."""
        def point_set(label):
            n = data.draw(st.integers(1, 12), label=label)
            return np.array(data.draw(st.lists(st.tuples(st.floats(-50, 50), st.floats(-50, 50)),
                                               min_size=n, max_size=n), label=label + "_pts"))
        a, b, c = point_set("a"), point_set("b"), point_set("c")
        hab = gm.hausdorff(a, b)
        assert hab == gm.hausdorff(b, a)
        assert gm.hausdorff(a, a) == 0.0
        assert gm.hausdorff(a, c) <= hab + gm.hausdorff(b, c) + 1e-9
        assert hab == orc.hausdorff(a, b)
