"""GPU pseudo-labelling against the reference's own
pseudo_label output on the same PNG directory (tests/golden/make_golden_labels.py).
Bar: the same files, ids, frame numbers, sources and full-frame decisions;
circle parameters within 1e-3 px; the CSV is compared after
parsing for the same reason."""

import hashlib
import logging

import numpy as np
import pytest

from paper_2210_14771_b200 import labels
from support import synth

from ._fixtures import load_json

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def frame_dir(tmp_path_factory):
    g = load_json("labels.json")
    d = tmp_path_factory.mktemp("frames")
    specs = synth.bench_specs(len(g["sha256"]), g["w"], g["h"], seed=g["spec_seed"])
    for k, (_, s) in enumerate(specs):
        f = synth.render(s, g["rng_seed0"] + k)
        assert hashlib.sha256(f.tobytes()).hexdigest() == g["sha256"][k], k
        labels.save_image(f, d / f"frame_{k:04d}.png")
    (d / "frame_0004b.png").write_bytes(b"not an image")
    (d / "notes.txt").write_text("ignored")
    return d


def _kw(kw):
    kw = dict(kw)
    if "source" in kw:
        kw["source"] = labels.Source(kw["source"])
    return kw


@pytest.mark.parametrize("case", ["all", "fps1", "seed7"])
@pytest.mark.parametrize("chunk", [256, 2])
def test_pseudo_label_matches_reference(frame_dir, case, chunk, caplog):
    want = load_json("labels.json")[case]
    with caplog.at_level(logging.WARNING):
        got = labels.pseudo_label(frame_dir, chunk=chunk, **_kw(want["kw"]))
    if case != "fps1":   # the unreadable file is sampled (and skipped) unless strided out
        assert "skipping unreadable frame" in caplog.text
    assert len(got) == len(want["anns"])
    for a, (sid, src, vno, fno, area, path) in zip(got, want["anns"]):
        assert (a.sample_id, a.source.value, a.video_no, a.frame_no, a.image_path) == \
            (sid, src, vno, fno, path)
        assert (a.area is None) == (area is None), (a, area)
        if area is not None:
            assert np.abs(np.array([a.area.cx, a.area.cy, a.area.r]) - area).max() <= 1e-3
