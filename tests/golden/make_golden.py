"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``eca`` from /root/reference/pkg/src (read-only; the bytecode cache
is disabled), runs the reference functions on deterministic inputs and writes
small JSON / NPZ fixtures next to this file.  Frames are not stored: each case
stores its recipe plus the SHA-256 of the reference's rendered bytes, and the
tests re-render with ``paper_2210_14771_b200.synth`` and check the hash first.
Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import math
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import eca  # noqa: E402
from eca import dataset as ds  # noqa: E402
from eca import edgenet as en  # noqa: E402
from eca import fitting as ft  # noqa: E402
from eca import handcrafted as hc  # noqa: E402
from eca import strips as st  # noqa: E402

OUT = Path(__file__).resolve().parent
CFG = eca.config_default()


# ---------------------------------------------------------------- recipes ---
def spec_to_dict(spec):
    d = dataclasses.asdict(spec)
    return d


def recipe_spec(spec, seed):
    return {"kind": "spec", "spec": spec_to_dict(spec), "seed": seed}


def make_frame(rec):
    k = rec["kind"]
    if k == "spec":
        s = dict(rec["spec"])
        if s["circle"] is not None:
            s["circle"] = eca.Circle(**s["circle"])
        if s["bleed"] is not None:
            s["bleed"] = ds.BleedSpot(**s["bleed"])
        if s["overlay"] is not None:
            s["overlay"] = ds.BoxOverlay(**s["overlay"])
        return ds.render_synthetic(ds.SyntheticSpec(**s), rec["seed"])[0]
    if k == "zeros":
        return np.zeros((rec["h"], rec["w"], 3), dtype=np.uint8)
    if k == "uniform":
        return np.full((rec["h"], rec["w"], 3), rec["value"], dtype=np.uint8)
    if k == "randint":
        return np.random.default_rng(rec["seed"]).integers(
            rec["lo"], rec["hi"], (rec["h"], rec["w"], 3)).astype(np.uint8)
    if k == "step":   # test_handcrafted.py:127-132
        rng = np.random.default_rng(rec["seed"])
        f = np.zeros((rec["h"], rec["w"], 3), dtype=np.uint8)
        b = rec["bright"]
        f[:, rec["step"]:, :] = rng.integers(b - 30, b + 30, (rec["h"], rec["w"] - rec["step"], 1))
        return f
    if k == "flip":
        return np.ascontiguousarray(make_frame(rec["base"])[:, ::-1, :])
    raise ValueError(k)


def sha(frame):
    return hashlib.sha256(np.ascontiguousarray(frame).tobytes()).hexdigest()


def fit_tuple(fit):
    if isinstance(fit, ft.Accepted):
        return [0, fit.circle.cx, fit.circle.cy, fit.circle.r, fit.score, fit.inlier_count]
    code = {ft.RejectionReason.NO_CANDIDATES: 1, ft.RejectionReason.LOW_SCORE: 2,
            ft.RejectionReason.GEOMETRY_GATE: 3}[fit.reason]
    return [code, 0.0, 0.0, 0.0, 0.0, 0]


def frame_case(name, rec, keep_scores=False, cfg=CFG, seed=0):
    frame = make_frame(rec)
    rows, size = eca.estimator.score_frame_strips(frame, eca.HANDCRAFTED, cfg)
    cands = [r.left_best for r in rows] + [r.right_best for r in rows]
    kept = ft.filter_candidates(cands, size, cfg)
    fit = ft.ransac_fit(kept, size, cfg, seed)
    area = eca.estimate(frame, eca.HANDCRAFTED, cfg, seed)
    case = {
        "name": name, "recipe": rec, "sha256": sha(frame), "seed": seed,
        "rows": st.strip_heights(frame.shape[0], cfg.strip_count, cfg.strip_weighting),
        "cand_x": [c.x for c in cands], "cand_y": [c.y for c in cands],
        "cand_score": [c.score for c in cands],
        "kept": [c in kept for c in cands],
        "fit": fit_tuple(fit),
        "estimate": None if isinstance(area, eca.FullFrame) else
        [area.circle.cx, area.circle.cy, area.circle.r, area.score],
    }
    scores = np.stack([r.scores for r in rows]) if keep_scores else None
    return case, scores


def main():
    # ------------------------------------------------------------ strips ---
    strip_cases = []
    for h in [14, 15, 16, 20, 40, 100, 240, 257, 480, 540, 720, 1000, 1080, 1081, 2160, 4320]:
        for s in [4, 7, 16, 17, 32, 64]:
            for a in [0.5, 4.0, 8.0, 13.3]:
                strip_cases.append({"H": h, "S": s, "alpha": a,
                                    "rows": st.strip_heights(h, s, a)})
    (OUT / "strip_rows.json").write_text(json.dumps(strip_cases))

    # ---------------------------------------------------------- triplets ---
    trip = {}
    for seed in [0, 1, 2, 3, 5, 9, 77, 1234, 2**31 - 1]:
        for att in [32]:
            for n in range(3, 65):
                trip[f"s{seed}_a{att}_n{n}"] = ft._sample_triplets(n, att, seed).astype(np.int16)
    for att in [1, 7, 100]:
        for n in [3, 4, 17, 32]:
            trip[f"s0_a{att}_n{n}"] = ft._sample_triplets(n, att, 0).astype(np.int16)
    np.savez_compressed(OUT / "triplets.npz", **trip)

    # ------------------------------------------------------------ render ---
    renders = []
    golden_spec = ds.SyntheticSpec(width=320, height=240, circle=eca.Circle(160.0, 120.0, 90.0),
                                   border_noise_sigma=2.0, content_brightness=150,
                                   bleed=ds.BleedSpot(30.0, 15.0, 200),
                                   overlay=ds.BoxOverlay(0, 0, 60, 24, 80))
    renders.append({"recipe": recipe_spec(golden_spec, 4242), "sha256": make_sha(golden_spec, 4242)})
    for w, h, sd in [(320, 240, 11), (960, 540, 3)]:
        for k, (cat, spec) in enumerate(ds.benchmark_specs(10, w, h, seed=sd)):
            renders.append({"recipe": recipe_spec(spec, 100 + k), "category": cat,
                            "sha256": make_sha(spec, 100 + k)})
    c2_specs = ds.benchmark_specs(40, 1920, 1080, seed=2024)
    (OUT / "c2_specs.json").write_text(json.dumps(
        [{"category": c, "spec": spec_to_dict(s)} for c, s in c2_specs]))
    (OUT / "render.json").write_text(json.dumps(renders))

    # ------------------------------------------------------- frame cases ---
    cases, score_arrays = [], {}

    def add(name, rec, keep=False, **kw):
        case, sc = frame_case(name, rec, keep, **kw)
        cases.append(case)
        if sc is not None:
            score_arrays[name] = sc

    add("golden_spec", recipe_spec(golden_spec, 4242), keep=True)
    for k, (cat, spec) in enumerate(ds.benchmark_specs(10, 320, 240, seed=11)):
        add(f"b320_{k}_{cat}", recipe_spec(spec, 100 + k), keep=True)
    for k, (cat, spec) in enumerate(ds.benchmark_specs(10, 640, 480, seed=5)):
        add(f"b640_{k}_{cat}", recipe_spec(spec, 200 + k), keep=(k < 5))
    clean = ds.benchmark_spec("clean", np.random.default_rng(7), 640, 480)
    add("conftest_clean", recipe_spec(clean, 123), keep=True)
    add("conftest_clean_flip", {"kind": "flip", "base": recipe_spec(clean, 123)}, keep=True)
    add("conftest_clean_seed5", recipe_spec(clean, 123), seed=5)
    add("centered_045", recipe_spec(ds.SyntheticSpec(640, 480, eca.Circle(319.5, 239.5, 0.45 * 640)), 8))
    add("oversized", recipe_spec(ds.SyntheticSpec(640, 480, eca.Circle(319.5, 239.5, 0.95 * 640),
                                                  adversarial=True), 5))
    add("uniform128", {"kind": "uniform", "h": 480, "w": 640, "value": 128}, keep=True)
    add("uniform90", {"kind": "uniform", "h": 480, "w": 640, "value": 90})
    add("zeros", {"kind": "zeros", "h": 480, "w": 640}, keep=True)
    add("white", {"kind": "uniform", "h": 64, "w": 64, "value": 255}, keep=True)
    add("noise_128x60", {"kind": "randint", "h": 60, "w": 128, "lo": 0, "hi": 256, "seed": 11}, keep=True)
    add("noise_129x61", {"kind": "randint", "h": 61, "w": 129, "lo": 0, "hi": 256, "seed": 2}, keep=True)
    add("step_400x100", {"kind": "step", "h": 100, "w": 400, "step": 100, "bright": 200, "seed": 3}, keep=True)
    add("min_8x14", {"kind": "randint", "h": 14, "w": 8, "lo": 0, "hi": 256, "seed": 4}, keep=True)
    add("odd_9x15", {"kind": "randint", "h": 15, "w": 9, "lo": 0, "hi": 256, "seed": 5}, keep=True)
    add("odd_333x257", recipe_spec(ds.benchmark_spec("clean", np.random.default_rng(9), 333, 257), 9), keep=True)
    add("dark_noise_640", {"kind": "randint", "h": 480, "w": 640, "lo": 0, "hi": 12, "seed": 3}, keep=True)
    dark = ds.benchmark_spec("dark", np.random.default_rng(0), 640, 480)
    add("dark_640", recipe_spec(dark, 3), keep=True)
    for k, (cat, spec) in enumerate(ds.benchmark_specs(5, 960, 540, seed=3)):
        add(f"b960_{k}_{cat}", recipe_spec(spec, 100 + k))
    # non-default configs on one frame
    for j, cfg in enumerate([dataclasses.replace(CFG, strip_count=8),
                             dataclasses.replace(CFG, strip_count=24, strip_weighting=4.0),
                             dataclasses.replace(CFG, gradient_threshold=35.0, angle_threshold_deg=20.0,
                                                 intensity_threshold=40.0),
                             dataclasses.replace(CFG, edge_margin_px=0, min_point_score=0.2),
                             dataclasses.replace(CFG, ransac_attempts=7, ransac_iterations=1),
                             dataclasses.replace(CFG, ransac_attempts=100, ransac_iterations=5)]):
        case, sc = frame_case(f"cfg{j}", recipe_spec(clean, 123), True, cfg=cfg)
        case["cfg"] = dataclasses.asdict(cfg)
        cases.append(case)
        score_arrays[f"cfg{j}"] = sc
    # BASELINE configs (1080p C1, C2 head, C4 4K edge cases)
    c1 = ds.benchmark_spec("clean", np.random.default_rng(0), 1920, 1080)
    add("c1_1080p", recipe_spec(c1, 0), keep=True)
    for k in range(10):
        add(f"c2_{k}_{c2_specs[k][0]}", recipe_spec(c2_specs[k][1], 30000 + k))
    W, H = 3840, 2160
    c0x, c0y = (W - 1) / 2.0, (H - 1) / 2.0
    add("c4_full_circle", recipe_spec(ds.SyntheticSpec(W, H, eca.Circle(c0x, c0y, 0.26 * W)), 7))
    add("c4_rectangle", recipe_spec(ds.SyntheticSpec(W, H, None), 7))
    add("c4_zeros", {"kind": "zeros", "h": H, "w": W})
    add("c4_uniform128", {"kind": "uniform", "h": H, "w": W, "value": 128})
    add("c4_dark_noise", {"kind": "randint", "h": H, "w": W, "lo": 0, "hi": 12, "seed": 3})
    add("c4_heavy_noise", recipe_spec(ds.SyntheticSpec(W, H, eca.Circle(c0x + 100, c0y - 50, 0.38 * W),
                                                       border_noise_sigma=12,
                                                       overlay=ds.BoxOverlay(0, 0, 843, 258, 90)), 7))
    (OUT / "frames.json").write_text(json.dumps(cases))
    np.savez_compressed(OUT / "scores.npz", **score_arrays)

    # -------------------------------------------------------------- fits ---
    rng = np.random.default_rng(2718)
    fits = []

    def fit_case(xs, ys, ss, w, h, seed, cfg=CFG, exhaustive=False, center=None):
        cands = [eca.EdgeCandidate(int(x), int(y), float(s), eca.Side.LEFT) for x, y, s in zip(xs, ys, ss)]
        fit = ft.ransac_fit(cands, (w, h), cfg, seed, exhaustive=exhaustive, center=center)
        fits.append({"x": [int(v) for v in xs], "y": [int(v) for v in ys], "s": [float(v) for v in ss],
                     "w": w, "h": h, "seed": seed, "exhaustive": exhaustive, "center": center,
                     "cfg": dataclasses.asdict(cfg), "fit": fit_tuple(fit)})

    for t in range(400):
        w, h = int(rng.integers(64, 2000)), int(rng.integers(64, 1200))
        kind = t % 4
        if kind == 0:      # uniform random points
            n = int(rng.integers(0, 33))
            xs, ys = rng.integers(0, w, n), rng.integers(0, h, n)
            ss = rng.uniform(0, 1, n)
        else:              # noisy circle + outliers
            cx = (w - 1) / 2 + rng.uniform(-0.25, 0.25) * w
            cy = (h - 1) / 2 + rng.uniform(-0.25, 0.25) * w
            r = rng.uniform(0.05, 0.9) * w
            n_in = int(rng.integers(2, 30))
            th = rng.uniform(0, 2 * np.pi, n_in)
            xs = np.round(cx + r * np.cos(th) + rng.normal(0, 1.0 * kind, n_in))
            ys = np.round(cy + r * np.sin(th) + rng.normal(0, 1.0 * kind, n_in))
            n_out = int(rng.integers(0, 6))
            xs = np.concatenate([xs, rng.integers(0, w, n_out)])
            ys = np.concatenate([ys, rng.integers(0, h, n_out)])
            ss = rng.uniform(0.03, 1.0, len(xs))
        seed = int(rng.integers(0, 2**31))
        fit_case(xs, ys, ss, w, h, seed)
    # exhaustive, center override, config variants
    for t in range(20):
        w, h = 640, 480
        n = int(rng.integers(3, 14))
        th = rng.uniform(0, 2 * np.pi, n)
        xs = np.round(319.5 + 20 + 190 * np.cos(th))
        ys = np.round(239.5 - 10 + 190 * np.sin(th))
        ss = rng.uniform(0.3, 1.0, n)
        fit_case(xs, ys, ss, w, h, t, exhaustive=True)
        fit_case(xs + 37, ys - 12, ss, w, h, t, center=(319.5 + 37, 239.5 - 12))
        fit_case(xs, ys, ss, w, h, t, cfg=dataclasses.replace(CFG, ransac_attempts=64, ransac_iterations=2,
                                                               min_circle_score=2.0,
                                                               min_circle_score_absolute=True))
    # reference test scenarios (test_fitting.py)
    truth = eca.Circle(320.0, 240.0, 100.0)
    offs = [(100, 0), (-100, 0), (0, 100), (0, -100), (60, 80), (-60, 80), (60, -80), (-60, -80),
            (80, 60), (-80, 60), (80, -60), (-80, -60)]
    fit_case([truth.cx + a for a, _ in offs], [truth.cy + b for _, b in offs], [0.9] * 12, 640, 480, 0)
    g = eca.Circle(319.5 + 20, 239.5 - 10, 0.3 * 640)
    th = np.linspace(0, 2 * math.pi, 16, endpoint=False)
    fit_case(np.round(g.cx + g.r * np.cos(th)), np.round(g.cy + g.r * np.sin(th)), [0.002] * 16, 640, 480, 1)
    big = eca.Circle(319.5, 239.5, 0.9 * 640)
    th = np.linspace(2.1, 2.6, 12)
    fit_case(np.round(big.cx + big.r * np.cos(th)), np.round(big.cy + big.r * np.sin(th)), [0.9] * 12, 640, 480, 0)
    (OUT / "fits.json").write_text(json.dumps(fits))

    # ----------------------------------------------------------- learned ---
    norm = en.ChannelStats(np.array([100.0] * 3), np.array([50.0] * 3))
    net = en.EdgeNet(norm, seed=0)
    learned = {}
    lcases = []
    for name, rec in [("clean640", recipe_spec(clean, 123)),
                      ("b320_0", recipe_spec(ds.benchmark_specs(1, 320, 240, seed=11)[0][1], 100)),
                      ("noise_128x60", {"kind": "randint", "h": 60, "w": 128, "lo": 0, "hi": 256, "seed": 11})]:
        frame = make_frame(rec)
        hs = st.strip_heights(frame.shape[0], CFG.strip_count, CFG.strip_weighting)
        rows = en.score_strips_learned(net, frame, hs)
        learned[name] = np.stack([r.scores for r in rows])
        cands = [r.left_best for r in rows] + [r.right_best for r in rows]
        kept = ft.filter_candidates(cands, (frame.shape[1], frame.shape[0]), CFG)
        fit = ft.ransac_fit(kept, (frame.shape[1], frame.shape[0]), CFG, 0)
        lcases.append({"name": name, "recipe": rec, "sha256": sha(frame),
                       "cand_x": [c.x for c in cands], "cand_score": [c.score for c in cands],
                       "fit": fit_tuple(fit)})
    for i, layer in enumerate(net.layers):
        learned[f"w{i}"] = layer.kernel
        learned[f"b{i}"] = layer.bias
    learned["blob"] = np.frombuffer(en.save_weights(net), dtype=np.uint8)
    np.savez_compressed(OUT / "learned.npz", **learned)
    (OUT / "learned.json").write_text(json.dumps(lcases))

    # -------------------------------------------------------------- crop ---
    crops = []
    rng = np.random.default_rng(31)
    for t in range(300):
        w, h = int(rng.integers(20, 2000)), int(rng.integers(20, 1200))
        c = eca.Circle(float(rng.uniform(-0.2, 1.2) * w), float(rng.uniform(-0.2, 1.2) * h),
                       float(rng.uniform(1.0, 1.0 * max(w, h))))
        ann = ds.EcaAnnotation("s", ds.Source.SYNTHETIC, 0, 0, c, "")
        xx, yy = np.meshgrid(np.arange(w), np.arange(h))
        frame = np.stack([xx & 255, (xx >> 8) | ((yy >> 8) << 4), yy & 255], axis=-1).astype(np.uint8)
        out = ds.crop_augment(ann, frame)
        bounds = None
        if out is not None:
            crop = out[0]
            p = crop[0, 0].astype(int)
            x0 = int(p[0] | ((p[1] & 15) << 8))
            y0 = int(p[2] | ((p[1] >> 4) << 8))
            bounds = [x0, y0, x0 + crop.shape[1] - 1, y0 + crop.shape[0] - 1]
            assert np.array_equal(frame[y0:bounds[3] + 1, x0:bounds[2] + 1], crop)
        crops.append({"w": w, "h": h, "circle": [c.cx, c.cy, c.r], "bounds": bounds})
    (OUT / "crops.json").write_text(json.dumps(crops))
    print("golden fixtures written to", OUT)


def make_sha(spec, seed):
    return sha(ds.render_synthetic(spec, seed)[0])


if __name__ == "__main__":
    main()
