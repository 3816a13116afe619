"""Memory-safety and race checks that stand in for compute-sanitizer (closed
on the GPU pool):

* canary zones: every output the handcrafted / learned / mask / crop kernels
  write is the middle of a larger buffer whose guard zones are filled with a
  pattern; after the launches the zones must be untouched;
* launch-shape determinism: the pipelined records must be bit-identical for
  every CTA shape / CTA cap / fit CTA width the launchers can pick (a race on
  tickets, survivor slots, the set guard or shared memory shows up as a
  difference between shapes), and across repeated runs.

The ECA_CHECKED build (tools/checked.sh) adds device-side index checks."""

import ctypes
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import _lib, api
from support import synth

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
PAT = 0xA5


def _guarded(n_bytes, dtype, shape, pad=4096):
    """(buffer, view): view of `shape` in the middle of a pattern-filled buffer."""
    itemsize = torch.empty((), dtype=dtype).element_size()
    buf = torch.full((pad + n_bytes + pad,), PAT, dtype=torch.uint8, device="cuda")
    view = buf[pad:pad + n_bytes].view(dtype).view(shape)
    assert n_bytes == int(np.prod(shape)) * itemsize
    return buf, view


def _zones_intact(buf, n_bytes, pad=4096):
    b = buf.cpu().numpy()
    return (b[:pad] == PAT).all() and (b[pad + n_bytes:] == PAT).all()


def _frames(n, w, h, seed=2024, rs=30000):
    specs = synth.bench_specs(n, w, h, seed=seed)
    return np.stack([synth.render(s, rs + k) for k, (_, s) in enumerate(specs)])


@pytest.mark.parametrize("w,h,b", [(640, 480, 20), (1920, 1080, 24), (333, 241, 17)])
def test_canary_zones_handcrafted(w, h, b):
    frames = torch.from_numpy(_frames(b, w, h)).cuda()
    eng = eb.ContentAreaEngine(h, w, b)
    want = eng.run(frames).clone()
    s = eng.n_strips
    lib = _lib.load()
    st = api._stream(eng.device)
    bx, xs = _guarded(b * 2 * s * 4, torch.int32, (b, 2 * s))
    by, ys = _guarded(b * 2 * s * 4, torch.int32, (b, 2 * s))
    bs, sc = _guarded(b * 2 * s * 8, torch.float64, (b, 2 * s))
    br, rec = _guarded(b * 40, torch.float64, (b, 5))
    n = ctypes.c_int64()
    lib.eca_points_workspace_bytes(b, s, ctypes.byref(n))
    bw, ws = _guarded(n.value, torch.uint8, (n.value,))
    ws.zero_()
    for _ in range(3):   # batched path: bounds + fit (rescore stage)
        _lib.check(lib.eca_estimate_batch_handcrafted(
            ctypes.c_void_p(frames.data_ptr()), b, frames.stride(0), frames.stride(1), eng._rows, None, s,
            ctypes.byref(eng.params), api._ptr(eng.trip), api._ptr(ws), api._ptr(xs), api._ptr(ys),
            api._ptr(sc), api._ptr(rec), None, 0, st), "estimate_batch")
    torch.cuda.synchronize()
    assert torch.equal(rec, want)
    bc, cnt = _guarded(64 * 4, torch.int32, (64,))
    cnt.zero_()
    _lib.check(lib.eca_estimate_handcrafted(   # latency path: in-warp rescore + fit
        ctypes.c_void_p(frames.data_ptr()), 16, frames.stride(0), frames.stride(1), eng._rows, None, s,
        ctypes.byref(eng.params), api._ptr(eng.trip), api._ptr(cnt), api._ptr(xs), api._ptr(ys), api._ptr(sc),
        api._ptr(rec), st), "estimate")
    torch.cuda.synchronize()
    assert torch.equal(rec[:16], want[:16])
    assert (cnt.cpu() == 0).all()
    for buf, nb in ((bx, b * 2 * s * 4), (by, b * 2 * s * 4), (bs, b * 2 * s * 8), (br, b * 40),
                    (bw, n.value), (bc, 256)):
        assert _zones_intact(buf, nb)


def test_canary_zones_mask_crop_learned():
    w, h, b = 640, 480, 6
    frames = torch.from_numpy(_frames(b, w, h)).cuda()
    eng = eb.ContentAreaEngine(h, w, b)
    rec = eng.run(frames).clone()
    lib = _lib.load()
    st = api._stream(eng.device)
    bm, masks = _guarded(b * h * w, torch.uint8, (b, h, w))
    _lib.check(lib.eca_draw_mask(api._ptr(rec), b, h, w, api._ptr(masks), h * w, st), "mask")
    torch.cuda.synchronize()
    assert _zones_intact(bm, b * h * w)
    bounds = torch.empty((b, 4), dtype=torch.int32, device="cuda")
    _lib.check(lib.eca_crop_bounds(api._ptr(rec), b, h, w, api._ptr(bounds), st), "crop_bounds")
    bh = bounds.cpu().numpy()
    sizes = [(0 if r[0] < 0 else (r[2] - r[0] + 1) * (r[3] - r[1] + 1) * 3) for r in bh]
    offs = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]), dtype=torch.int64, device="cuda")
    total = int(sum(sizes))
    bo, out = _guarded(total, torch.uint8, (total,))
    _lib.check(lib.eca_crop_copy(ctypes.c_void_p(frames.data_ptr()), b, frames.stride(0), frames.stride(1),
                                 api._ptr(bounds), api._ptr(offs), api._ptr(out),
                                 int(max(r[3] - r[1] + 1 for r in bh if r[0] >= 0)), st), "crop_copy")
    torch.cuda.synchronize()
    assert _zones_intact(bo, total)
    net = eb.EdgeNet(eb.ChannelStats([100.0] * 3, [50.0] * 3), seed=0)
    le = eb.ContentAreaEngine(h, w, b, variant=eb.Learned(net))
    s = le.n_strips
    bp, probs = _guarded(b * s * (w - 6) * 4, torch.float32, (b, s, w - 6))
    for flags in (0, _lib.LEARNED_SIMT):
        _lib.check(lib.eca_points_learned_ex(
            ctypes.c_void_p(frames.data_ptr()), b, frames.stride(0), frames.stride(1), le._rows, None, s, h, w,
            api._ptr(le.w_dev), le.norm, flags, api._ptr(probs), api._ptr(le.xs), api._ptr(le.ys),
            api._ptr(le.sc), st), "learned")
        torch.cuda.synchronize()
        assert _zones_intact(bp, b * s * (w - 6) * 4)


_SHAPE_SCRIPT = r"""
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb
from support import synth
specs = synth.bench_specs(40, 960, 540, seed=2024)
frames = torch.from_numpy(np.stack([synth.render(s, 33000 + k) for k, (_, s) in enumerate(specs)])).cuda()
B = 24
pool = frames[[k % 40 for k in range(5 * B)]].contiguous()
eng = eb.ContentAreaEngine(540, 960, B)
out = []
for rep in range(3):
    recs = eng.run_stream(pool, rep, 9)
    eng.fence()
    torch.cuda.synchronize()
    out += [r.clone() for r in recs]
out.append(eng.run(pool[:B]).clone())
torch.save([o.cpu() for o in out], sys.argv[1])
"""


def test_launch_shapes_are_deterministic(tmp_path):
    """The same stream under every launch shape the launchers can pick gives
    bit-identical records (tickets, slots, guard and smem are race-free)."""
    script = tmp_path / "shape.py"
    script.write_text(_SHAPE_SCRIPT)
    results = {}
    for env in ({}, {"ECA_BWARPS": "1"}, {"ECA_BWARPS": "2"}, {"ECA_BWARPS": "8"}, {"ECA_BCTAS": "1"},
                {"ECA_FIT_FPB": "1"}, {"ECA_FIT_FPB": "3"}, {"ECA_PIPE_SHARE": "0"}):
        out = tmp_path / f"r{len(results)}.pt"
        r = subprocess.run([sys.executable, str(script), str(out)], cwd=ROOT, env={**os.environ, **env},
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, (env, r.stderr[-2000:])
        results[str(env)] = torch.load(out)
    ref = results["{}"]
    for k, v in results.items():
        assert len(v) == len(ref)
        for a, b in zip(v, ref):
            assert torch.equal(a, b), k
