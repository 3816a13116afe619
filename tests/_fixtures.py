"""Rebuild golden-fixture frames from their recipes (no /root/reference needed)."""

from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from support import synth
from paper_2210_14771_b200.params import EcaConfig
from paper_2210_14771_b200.shapes import Circle

GOLDEN = Path(__file__).resolve().parent / "golden"


def load_json(name):
    return json.loads((GOLDEN / name).read_text())


@lru_cache(maxsize=None)
def load_npz(name):
    return dict(np.load(GOLDEN / name))


def spec_from_dict(d):
    d = dict(d)
    if d["circle"] is not None:
        d["circle"] = Circle(**d["circle"])
    if d["bleed"] is not None:
        d["bleed"] = synth.BleedSpot(**d["bleed"])
    if d["overlay"] is not None:
        d["overlay"] = synth.BoxOverlay(**d["overlay"])
    return synth.SyntheticSpec(**d)


def make_frame(rec):
    k = rec["kind"]
    if k == "spec":
        return synth.render(spec_from_dict(rec["spec"]), rec["seed"])
    if k == "zeros":
        return np.zeros((rec["h"], rec["w"], 3), dtype=np.uint8)
    if k == "uniform":
        return np.full((rec["h"], rec["w"], 3), rec["value"], dtype=np.uint8)
    if k == "randint":
        return np.random.default_rng(rec["seed"]).integers(
            rec["lo"], rec["hi"], (rec["h"], rec["w"], 3)).astype(np.uint8)
    if k == "step":
        rng = np.random.default_rng(rec["seed"])
        f = np.zeros((rec["h"], rec["w"], 3), dtype=np.uint8)
        b = rec["bright"]
        f[:, rec["step"]:, :] = rng.integers(b - 30, b + 30, (rec["h"], rec["w"] - rec["step"], 1))
        return f
    if k == "flip":
        return np.ascontiguousarray(make_frame(rec["base"])[:, ::-1, :])
    if k == "osd":   # tests/golden/make_golden_configs.py
        return synth.stamp_osd_text(make_frame(rec["base"]), rec["seed"])
    raise ValueError(k)


def sha(frame):
    return hashlib.sha256(np.ascontiguousarray(frame).tobytes()).hexdigest()


def case_cfg(case):
    return EcaConfig(**case["cfg"]) if "cfg" in case else EcaConfig()


def frame_cases(max_pixels=None):
    cases = load_json("frames.json")
    if max_pixels is not None:
        cases = [c for c in cases if _pixels(c["recipe"]) <= max_pixels]
    return cases


def _pixels(rec):
    if rec["kind"] == "spec":
        return rec["spec"]["width"] * rec["spec"]["height"]
    if rec["kind"] in ("flip", "osd"):
        return _pixels(rec["base"])
    return rec["w"] * rec["h"]
