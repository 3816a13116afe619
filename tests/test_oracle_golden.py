"""Pin the CPU oracle (and the synthetic renderer) to the reference's own outputs.

Fixtures in tests/golden were produced by running the reference package
(make_golden.py).  Everything here runs on CPU.
"""

import math

import numpy as np
import pytest

from oracle import eca_oracle as orc
from support import synth
from paper_2210_14771_b200.params import EcaConfig

from ._fixtures import case_cfg, frame_cases, load_json, load_npz, make_frame, sha, spec_from_dict

SMALL = 700 * 500


def test_strip_rows_match_reference():
    for c in load_json("strip_rows.json"):
        assert orc.strip_rows(c["H"], c["S"], c["alpha"]) == c["rows"], c


def test_known_strip_rows_1080():
    # test_strips.py:8-14 (50-digit oracle)
    assert orc.strip_rows(1080, 16, 8.0) == [25, 40, 65, 103, 160, 241, 346, 473, 607, 734,
                                             839, 920, 977, 1015, 1040, 1055]


def test_renderer_golden_hashes():
    for r in load_json("render.json"):
        assert sha(make_frame(r["recipe"])) == r["sha256"]
    # dataset.py golden spec pinned by the reference's own test (test_dataset.py:39)
    assert load_json("render.json")[0]["sha256"] == \
        "cab24262a56c854112995e643ce9a24af27b04eba3b70e769a4d19010f62be86"


def test_bench_specs_match_reference():
    ref = load_json("c2_specs.json")
    mine = synth.bench_specs(len(ref), 1920, 1080, seed=2024)
    for (cat, spec), r in zip(mine, ref):
        assert cat == r["category"]
        assert spec == spec_from_dict(r["spec"])


@pytest.mark.parametrize("case", frame_cases(max_pixels=SMALL), ids=lambda c: c["name"])
def test_oracle_candidates_and_fit_small(case):
    frame = make_frame(case["recipe"])
    assert sha(frame) == case["sha256"]
    cfg = case_cfg(case)
    xs, ys, sc, rows, scores = orc.handcrafted_candidates(frame, cfg)
    assert rows == case["rows"]
    assert xs.tolist() == case["cand_x"]
    assert ys.tolist() == case["cand_y"]
    assert sc.tolist() == case["cand_score"]      # same numpy ops -> same bits
    npz = load_npz("scores.npz")
    if case["name"] in npz:
        assert np.array_equal(scores, npz[case["name"]])
    h, w = frame.shape[:2]
    keep = orc.keep_mask(xs, ys, sc, w, h, cfg)
    assert keep.tolist() == case["kept"]
    fit = orc.ransac(xs[keep], ys[keep], sc[keep], w, h, cfg, case["seed"])
    assert list(fit) == case["fit"]


@pytest.mark.slow
@pytest.mark.parametrize("case", [c for c in frame_cases() if c["name"].startswith(("c1", "c2_0", "c4_full", "c4_zeros"))],
                         ids=lambda c: c["name"])
def test_oracle_large_frames(case):
    frame = make_frame(case["recipe"])
    assert sha(frame) == case["sha256"]
    st, cx, cy, r, s, n = orc.estimate(frame, EcaConfig(), case["seed"])
    assert [st, cx, cy, r, s, n] == case["fit"]


@pytest.mark.parametrize("case", load_json("configs.json"), ids=lambda c: c["name"])
def test_oracle_config_cases(case):
    """Non-default configs (t_g 3/100/200, theta 5/90, t_i 5/200, a combo)
    and the 4K OSD-text frame: the oracle reproduces the reference's
    candidates, scores, filter and fit bit for bit."""
    frame = make_frame(case["recipe"])
    assert sha(frame) == case["sha256"]
    cfg = case_cfg(case)
    xs, ys, sc, rows, scores = orc.handcrafted_candidates(frame, cfg)
    assert rows == case["rows"]
    assert xs.tolist() == case["cand_x"] and ys.tolist() == case["cand_y"]
    assert sc.tolist() == case["cand_score"]
    npz = load_npz("configs_scores.npz")
    if case["name"] in npz:
        assert np.array_equal(scores, npz[case["name"]])
    h, w = frame.shape[:2]
    keep = orc.keep_mask(xs, ys, sc, w, h, cfg)
    assert keep.tolist() == case["kept"]
    assert list(orc.ransac(xs[keep], ys[keep], sc[keep], w, h, cfg, case["seed"])) == case["fit"]


def test_triplets_match_reference():
    for key, arr in load_npz("triplets.npz").items():
        seed, att, n = (int(p[1:]) for p in key.split("_"))
        assert np.array_equal(orc.sample_triplets(n, att, seed), arr), key


def test_fits_match_reference():
    for c in load_json("fits.json"):
        cfg = EcaConfig(**c["cfg"])
        center = tuple(c["center"]) if c["center"] is not None else None
        out = orc.ransac(c["x"], c["y"], c["s"], c["w"], c["h"], cfg, c["seed"],
                         exhaustive=c["exhaustive"], center=center)
        assert list(out) == c["fit"], c


def test_learned_matches_reference():
    npz = load_npz("learned.npz")
    layers = orc.glorot_layers(0)
    for i, (k, b) in enumerate(layers):
        assert np.array_equal(k, npz[f"w{i}"]) and np.array_equal(b, npz[f"b{i}"])
    cfg = EcaConfig()
    for c in load_json("learned.json"):
        frame = make_frame(c["recipe"])
        assert sha(frame) == c["sha256"]
        rows = orc.strip_rows(frame.shape[0], 16, 8.0)
        s = orc.learned_scores(frame, rows, [100.0] * 3, [50.0] * 3, layers)
        assert np.array_equal(s, npz[c["name"]])
        xs, ys, sc = orc.candidates_from_scores(s, rows)
        assert xs.tolist() == c["cand_x"] and sc.tolist() == c["cand_score"]
        h, w = frame.shape[:2]
        k = orc.keep_mask(xs, ys, sc, w, h, cfg)
        assert list(orc.ransac(xs[k], ys[k], sc[k], w, h, cfg, 0)) == c["fit"]


def test_crop_bounds_match_reference():
    for c in load_json("crops.json"):
        b = orc.crop_bounds(*c["circle"], c["w"], c["h"])
        assert (list(b) if b is not None else None) == c["bounds"], c


def test_disk_mask_matches_scalar_contains():
    # geometry.py:30-34 evaluated per pixel in Python floats
    for cx, cy, r in [(10.5, 7.25, 6.0), (0.0, 0.0, 3.0), (15.2, -2.0, 9.999)]:
        m = orc.disk_mask(cx, cy, r, 12, 20)
        for y in range(12):
            for x in range(20):
                dx, dy = x - cx, y - cy
                assert m[y, x] == (dx * dx + dy * dy <= r * r)


# ---- evaluation row: metrics.py restated in the oracle
def _circ(c):
    return None if c is None else tuple(c)


def test_oracle_boundary_points_match_reference():
    g, pts = load_json("metrics.json"), load_npz("metrics_points.npz")
    for i, c in enumerate(g["cases"]):
        bp = orc.boundary_points(_circ(c["pred"]), c["w"], c["h"], c["spacing"])
        bt = orc.boundary_points(_circ(c["truth"]), c["w"], c["h"], c["spacing"])
        assert (len(bp), len(bt)) == (c["n_pred"], c["n_truth"]), (i, c)
        if f"p{i}" in pts:
            assert np.array_equal(bp, pts[f"p{i}"]) and np.array_equal(bt, pts[f"t{i}"]), i


def test_oracle_hausdorff_matches_reference():
    g, pts = load_json("metrics.json"), load_npz("metrics_points.npz")
    for k, s in enumerate(g["sets"]):
        assert orc.hausdorff(pts[f"ha{k}"], pts[f"hb{k}"]) == s["hd"], k
    for i, c in enumerate(g["cases"]):
        if c["w"] > 640:
            continue   # the brute-force oracle is O(n^2): small frames here, all sizes on the GPU
        bp = orc.boundary_points(_circ(c["pred"]), c["w"], c["h"], c["spacing"])
        bt = orc.boundary_points(_circ(c["truth"]), c["w"], c["h"], c["spacing"])
        assert orc.hausdorff(bp, bt) == c["hd"], (i, c)
        if c["spacing"] == 1.0:
            assert orc.area_error_px(_circ(c["pred"]), _circ(c["truth"]), c["w"], c["h"]) == c["nh"]


# ---- learned training row: edgenet.py training restated in the oracle
def train_inputs(m=24, h=7, w=64, seed=5):
    """Same recipe as tests/golden/make_golden_train.py."""
    rng = np.random.default_rng(seed)
    x = rng.normal(0.0, 1.0, (m, 5, h, w)).astype(np.float32)
    t = rng.uniform(0.0, 1.0, (m, 1, h - 6, w - 6)).astype(np.float32)
    return x, t


def _pack(layers):
    return np.concatenate([np.concatenate([k.ravel(), b.ravel()]) for k, b in layers]).astype(np.float32)


def test_oracle_training_step_matches_reference():
    g = load_npz("train.npz")
    layers = orc.glorot_layers(0)
    assert np.array_equal(_pack(layers), g["w0"])
    x, t = train_inputs()
    logits, _ = orc.forward_logits(x[:8], layers)
    assert np.array_equal(logits, g["logits"])
    loss, grads, _ = orc.train_step(x[:8], t[:8], layers, 0.0)
    assert loss == g["loss"][0]
    assert np.array_equal(_pack(grads), g["grads"])


def test_oracle_train_loop_matches_reference():
    g = load_npz("train.npz")
    x, t = train_inputs()
    xv, tv = train_inputs(m=10, seed=6)
    best, tl, vl, be = orc.train(orc.glorot_layers(0), x, t, xv, tv, lr=0.05, batch=4, patience=2,
                                 epochs=6, seed=3)
    assert tl == g["train_losses"].tolist() and vl == g["val_losses"].tolist()
    assert be == g["best_epoch"][0]
    assert np.array_equal(_pack(best), g["w_trained"])
    best, tl, _, _ = orc.train(orc.glorot_layers(0), x, t, None, None, lr=0.02, batch=5, epochs=2,
                               shuffle=False)
    assert tl == g["train_losses_noval"].tolist()
    assert np.array_equal(_pack(best), g["w_noval"])
