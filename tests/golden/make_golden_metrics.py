"""Golden fixtures for the evaluation row, made by running the
REFERENCE's own metrics module (/root/reference/pkg/src/eca/metrics.py) in the
build container:

    python tests/golden/make_golden_metrics.py

Writes metrics.json (cases: areas, frame size, spacing, the reference's sample
counts, Hausdorff and normalised-Hausdorff values, evaluate_dataset reports)
and metrics_points.npz (the reference's boundary samples of the small cases).
Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from eca import metrics as M  # noqa: E402
from eca.geometry import FULL_FRAME, Circle  # noqa: E402

OUT = Path(__file__).resolve().parent


def area(c):
    return FULL_FRAME if c is None else Circle(*c)


def cases():
    out = []
    for w, h in ((100, 100), (300, 150), (640, 480), (1920, 1080), (3840, 2160)):
        cx, cy = (w - 1) / 2, (h - 1) / 2
        fixed = [
            ((cx, cy, 0.3 * h), (cx, cy, 0.33 * h)),             # concentric, interior
            ((cx, cy, 0.6 * h), (cx + 3, cy - 2, 0.6 * h + 5)),  # clipped top and bottom
            (None, (cx, cy, 0.55 * w)),                          # full frame vs clipped
            (None, None),                                         # both full frame
            ((cx, cy, 5.0 * w), None),                            # swallowing circle
            ((cx, cy, 0.3 * h), (cx, cy, 0.3 * h)),               # identical
            ((0.0, 0.0, 0.5 * h), (w - 1.0, h - 1.0, 0.5 * h)),  # corner circles
            ((cx, cy, cx), (cx, cy, cy)),                         # tangent to the edges
            ((-0.1 * w, cy, 0.4 * w), (cx, -0.2 * h, 0.5 * h)),  # centres outside
        ]
        for p, t in fixed:
            out.append((p, t, w, h, 1.0))
    rng = np.random.default_rng(2210)
    for k in range(60):
        w, h = [(640, 480), (1920, 1080), (300, 150), (3840, 2160)][k % 4]
        sp = [1.0, 0.5, 2.0, 1.0][k // 4 % 4]

        def rnd():
            if rng.random() < 0.1:
                return None
            while True:
                c = (float(rng.uniform(-0.2, 1.2) * w), float(rng.uniform(-0.2, 1.2) * h),
                     float(rng.uniform(0.05, 1.0) * max(w, h)))
                try:
                    M.boundary_points(Circle(*c), w, h)
                    return c
                except ValueError:
                    continue
        t = rnd()
        p = None if t is None or rng.random() < 0.2 else \
            (t[0] + float(rng.normal(0, 10)), t[1] + float(rng.normal(0, 10)), t[2] + float(rng.normal(0, 10)))
        out.append((p, t, w, h, sp))
    return out


def main():
    items, pts = [], {}
    for i, (p, t, w, h, sp) in enumerate(cases()):
        bp = M.boundary_points(area(p), w, h, sp)
        bt = M.boundary_points(area(t), w, h, sp)
        hd = M.hausdorff(bp, bt)
        nh = M.area_error_px(area(p), area(t), w, h) if sp == 1.0 else M.normalized_hausdorff(bp, bt, w, h)
        items.append({"pred": p, "truth": t, "w": w, "h": h, "spacing": sp,
                      "n_pred": len(bp), "n_truth": len(bt), "hd": hd, "nh": nh,
                      "len_pred": M.boundary_length(area(p), w, h),
                      "len_truth": M.boundary_length(area(t), w, h)})
        if w <= 300:
            pts[f"p{i}"], pts[f"t{i}"] = bp, bt
    # a circle that misses the frame: ValueError in the reference
    try:
        M.boundary_points(Circle(-500.0, -500.0, 10.0), 100, 100)
        raise SystemExit("expected ValueError")
    except ValueError as e:
        miss = str(e)
    # point-set Hausdorff cases (arbitrary sets)
    rng = np.random.default_rng(7)
    sets = []
    for k in range(12):
        a = rng.uniform(-50, 50, (int(rng.integers(1, 400)), 2))
        b = rng.uniform(-50, 50, (int(rng.integers(1, 400)), 2)) + (k % 3) * 10.0
        pts[f"ha{k}"], pts[f"hb{k}"] = a, b
        sets.append({"hd": M.hausdorff(a, b)})
    # evaluate_dataset over the 1080p cases
    sel = [it for it in items if it["w"] == 1920 and it["spacing"] == 1.0]
    preds = {f"s{i:03d}": area(it["pred"]) for i, it in enumerate(sel)}
    truths = {f"s{i:03d}": area(it["truth"]) for i, it in enumerate(sel)}
    rep = M.evaluate_dataset(preds, truths, (1920, 1080))
    report = {"ids": sorted(preds), "pred": [it["pred"] for it in sel], "truth": [it["truth"] for it in sel],
              "avg": rep.avg_error_px, "miss": rep.miss_pct, "bad": rep.bad_miss_pct,
              "labels": [s.label.value for s in rep.per_sample],
              "markdown": M.report_markdown({"handcrafted": rep})}
    (OUT / "metrics.json").write_text(json.dumps({"cases": items, "miss_message": miss,
                                                   "sets": sets, "report": report}))
    np.savez_compressed(OUT / "metrics_points.npz", **pts)
    print(f"{len(items)} area cases, {len(sets)} point-set cases, report over {len(sel)} samples")


if __name__ == "__main__":
    main()
