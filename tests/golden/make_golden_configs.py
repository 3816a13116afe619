"""Golden fixtures for NON-DEFAULT configs and the 4K OSD-text frame, produced
by running the REFERENCE package itself (same method as make_golden.py):

    python tests/golden/make_golden_configs.py

Writes configs.json (+ configs_scores.npz: every column score of the 640x480
cases).  The configs stretch the FP32 bound-and-prune prefilter of the
handcrafted kernels: gradient thresholds 3 / 100 / 200 (the tanh term's
cancellation grows with t_g), angle thresholds 5 / 90 deg, intensity
thresholds 5 (outside the FP32 envelope: the kernels fall back to exhaustive
FP64 scoring) and 200, and one combination.  The frames are the conftest
clean 640x480 render, the C1 1080p frame, two C2 1080p frames, and a C4 4K
frame with heavy border noise, a box overlay and burned-in OSD text
(support.synth.stamp_osd_text, applied to the reference's own render).
"""

from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent.parent))

import numpy as np  # noqa: E402

import make_golden as mg  # noqa: E402  (imports eca from /root/reference)
from make_golden import CFG, ds, eca, recipe_spec  # noqa: E402
from support import synth  # noqa: E402

CONFIGS = {
    "tg3": dict(gradient_threshold=3.0),
    "tg100": dict(gradient_threshold=100.0),
    "tg200": dict(gradient_threshold=200.0),
    "theta5": dict(angle_threshold_deg=5.0),
    "theta90": dict(angle_threshold_deg=90.0),
    "ti5": dict(intensity_threshold=5.0),
    "ti200": dict(intensity_threshold=200.0),
    "combo": dict(gradient_threshold=150.0, angle_threshold_deg=8.0, intensity_threshold=60.0),
}


_REF_MAKE_FRAME = mg.make_frame


def make_frame(rec):
    if rec["kind"] == "osd":
        return synth.stamp_osd_text(make_frame(rec["base"]), rec["seed"])
    return _REF_MAKE_FRAME(rec)


def main():
    mg.make_frame = make_frame   # frame_case renders through the osd-aware maker
    clean = ds.benchmark_spec("clean", np.random.default_rng(7), 640, 480)
    c1 = ds.benchmark_spec("clean", np.random.default_rng(0), 1920, 1080)
    c2 = ds.benchmark_specs(4, 1920, 1080, seed=2024)
    W, H = 3840, 2160
    c0x, c0y = (W - 1) / 2.0, (H - 1) / 2.0
    heavy = recipe_spec(ds.SyntheticSpec(W, H, eca.Circle(c0x + 100, c0y - 50, 0.38 * W),
                                         border_noise_sigma=12,
                                         overlay=ds.BoxOverlay(0, 0, 843, 258, 90)), 7)
    osd = {"kind": "osd", "base": heavy, "seed": 7}
    frames = [("clean640", recipe_spec(clean, 123), True),
              ("c1_1080p", recipe_spec(c1, 0), False),
              ("c2_1_dark", recipe_spec(c2[1][1], 30001), False),
              ("c2_3_overlay", recipe_spec(c2[3][1], 30003), False)]
    cases, scores = [], {}
    for cname, kw in [("default", {})] + list(CONFIGS.items()):
        cfg = dataclasses.replace(CFG, **kw)
        todo = frames if kw else []
        if cname in ("default", "tg100", "theta5", "ti5"):
            todo = todo + [("c4_osd_text", osd, False)]
        for fname, rec, keep in todo:
            name = f"{cname}_{fname}"
            case, sc = mg.frame_case(name, rec, keep, cfg=cfg)
            case["cfg"] = dataclasses.asdict(cfg)
            cases.append(case)
            if sc is not None:
                scores[name] = sc
            print(name, case["fit"][:1], flush=True)
    (HERE / "configs.json").write_text(json.dumps(cases))
    np.savez_compressed(HERE / "configs_scores.npz", **scores)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
