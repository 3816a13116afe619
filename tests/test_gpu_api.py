"""GPU tests of the public API's host-side behaviour: the cached single-frame
path, device selection, concurrent callers on different streams, odd host
strides and the per-frame error contract (estimator.py:55-111)."""

import threading

import numpy as np
import pytest
import torch

import paper_2210_14771_b200 as eb
from support import synth

pytestmark = pytest.mark.gpu


def _frames(n, w=640, h=480, seed=4):
    specs = synth.bench_specs(n, w, h, seed=seed)
    return np.stack([synth.render(s, 50 + k) for k, (_, s) in enumerate(specs)])


def test_single_frame_path_equals_batch_path():
    frames = _frames(6)
    want = eb.estimate_batch(torch.from_numpy(frames).cuda())
    for k, f in enumerate(frames):
        assert eb.estimate(f) == want[k]
        assert eb.estimate(torch.from_numpy(f).cuda()) == want[k]
        assert eb.estimate(torch.from_numpy(f)) == want[k]           # CPU tensor
        assert eb.estimate(f, device="cuda:0") == want[k]


def test_single_frame_path_strided_inputs():
    f = _frames(1)[0]
    want = eb.estimate(f)
    pad = np.zeros((480, 650, 3), dtype=np.uint8)
    pad[:, 5:645] = f
    assert eb.estimate(pad[:, 5:645]) == want                           # padded rows
    t = torch.zeros((480, 650, 3), dtype=torch.uint8, device="cuda")
    t[:, 5:645] = torch.from_numpy(f).cuda()
    assert eb.estimate(t[:, 5:645]) == want
    flip = np.ascontiguousarray(f[::-1])
    assert eb.estimate(f[::-1]) == eb.estimate(flip)                   # negative row stride
    assert eb.estimate_batch([f[::-1]]) == [eb.estimate(flip)]


def test_batch_reports_oversized_frames_per_index():
    f = _frames(1)[0]
    wide = np.zeros((20, eb.api._lib.MAX_WIDTH + 8, 3), dtype=np.uint8)
    out = eb.estimate_batch([f, wide, f])
    assert isinstance(out[1], eb.FrameError) and out[1].index == 1 and "too large" in out[1].message
    assert out[0] == out[2] == eb.estimate(f)


def test_concurrent_callers_on_separate_streams():
    """Two host threads, each on its own stream, running batched estimates
    (bounds + fit with per-(device, stream) workspaces) and single-frame
    estimates at the same time: every result equals the serial one."""
    frames = _frames(24, 960, 540, seed=9)
    dev = torch.from_numpy(frames).cuda()
    want_batch = eb.estimate_batch(dev)
    want_one = [eb.estimate(f) for f in frames[:6]]
    errors = []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    assert eb.estimate_batch(dev) == want_batch
                    assert [eb.estimate(f) for f in frames[:6]] == want_one
        except Exception as exc:  # noqa: BLE001
            errors.append((k, repr(exc)))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
