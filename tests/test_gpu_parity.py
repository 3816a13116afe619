"""GPU parity: the CUDA path against the reference's golden fixtures and the
CPU oracle on the same inputs.  Tolerances:
  candidates (x, y, side) exact; |d score| <= max(8 ulp, 1e-12)
  fit status + inlier count exact; cx, cy, r within 1e-3 px; score rel 1e-12
  masks / crop bounds bit-exact; learned probabilities within 1e-5.
"""

import numpy as np
import pytest
import torch

import paper_2210_14771_b200 as eb
from oracle import eca_oracle as orc
from support import synth

from ._fixtures import case_cfg, frame_cases, load_json, load_npz, make_frame, sha

pytestmark = pytest.mark.gpu

SCORE_ULPS = 8
SCORE_ABS = 1e-12
PX_TOL = 1e-3


def close_scores(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    tol = np.maximum(SCORE_ULPS * np.spacing(np.abs(b)), SCORE_ABS)
    return np.abs(a - b) <= tol


def assert_fit_equal(got, want, ctx=""):
    """got: FitResult; want: oracle tuple (status, cx, cy, r, score, inliers)."""
    st = want[0]
    if st == 0:
        assert isinstance(got, eb.Accepted), (ctx, got, want)
        assert abs(got.circle.cx - want[1]) <= PX_TOL, (ctx, got, want)
        assert abs(got.circle.cy - want[2]) <= PX_TOL, (ctx, got, want)
        assert abs(got.circle.r - want[3]) <= PX_TOL, (ctx, got, want)
        assert got.score == pytest.approx(want[4], rel=1e-12), (ctx, got, want)
        assert got.inlier_count == want[5], (ctx, got, want)
    else:
        code = {1: eb.RejectionReason.NO_CANDIDATES, 2: eb.RejectionReason.LOW_SCORE,
                3: eb.RejectionReason.GEOMETRY_GATE}[st]
        assert got == eb.Rejected(code), (ctx, got, want)


def fit_tuple_of_area(area):
    return area


SMALL = frame_cases(max_pixels=1000 * 600)


@pytest.mark.parametrize("case", SMALL, ids=lambda c: c["name"])
def test_candidates_match_reference(case):
    frame = make_frame(case["recipe"])
    assert sha(frame) == case["sha256"]
    cfg = case_cfg(case)
    pts = eb.get_points(frame, cfg=cfg)
    s = len(case["rows"])
    assert [p.x for p in pts] == case["cand_x"]
    assert [p.y for p in pts] == case["cand_y"]
    assert [p.side for p in pts] == [eb.Side.LEFT] * s + [eb.Side.RIGHT] * s
    assert close_scores([p.score for p in pts], case["cand_score"]).all()


@pytest.mark.parametrize("case", [c for c in SMALL if c["name"] in load_npz("scores.npz")],
                         ids=lambda c: c["name"])
def test_score_rows_match_reference(case):
    frame = make_frame(case["recipe"])
    rows, size = eb.score_frame_strips(frame, cfg=case_cfg(case))
    got = np.stack([r.scores for r in rows])
    want = load_npz("scores.npz")[case["name"]]
    assert size == (frame.shape[1], frame.shape[0])
    ok = close_scores(got, want)
    assert ok.all(), (np.argwhere(~ok)[:5], got[~ok][:5], want[~ok][:5])
    assert [r.left_best.x for r in rows] + [r.right_best.x for r in rows] == case["cand_x"]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: c["name"])
def test_estimate_matches_reference(case):
    frame = make_frame(case["recipe"])
    cfg = case_cfg(case)
    area = eb.estimate(frame, cfg=cfg, seed=case["seed"])
    if case["estimate"] is None:
        assert area == eb.FULL_FRAME
    else:
        assert isinstance(area, eb.CircularArea)
        cx, cy, r, s = case["estimate"]
        assert abs(area.circle.cx - cx) <= PX_TOL and abs(area.circle.cy - cy) <= PX_TOL
        assert abs(area.circle.r - r) <= PX_TOL
        assert area.score == pytest.approx(s, rel=1e-12)


def test_fits_match_reference():
    fails = []
    for i, c in enumerate(load_json("fits.json")):
        cfg = eb.EcaConfig(**c["cfg"])
        cands = [eb.EdgeCandidate(x, y, s, eb.Side.LEFT) for x, y, s in zip(c["x"], c["y"], c["s"])]
        center = tuple(c["center"]) if c["center"] is not None else None
        got = eb.ransac_fit(cands, (c["w"], c["h"]), cfg, c["seed"], exhaustive=c["exhaustive"],
                            center=center)
        try:
            assert_fit_equal(got, c["fit"], i)
        except AssertionError as e:
            fails.append(str(e)[:300])
    assert not fails, fails[:5]


@pytest.mark.parametrize("case", [c for c in frame_cases() if c not in SMALL], ids=lambda c: c["name"])
def test_large_frames_match_reference(case):
    """1080p (C1, C2 head) and 4K edge cases (C4) against the reference fixtures."""
    frame = make_frame(case["recipe"])
    assert sha(frame) == case["sha256"]
    t = torch.from_numpy(frame).cuda()
    pts = eb.get_points(t)
    assert [p.x for p in pts] == case["cand_x"]
    assert close_scores([p.score for p in pts], case["cand_score"]).all()
    fit = eb.fit_area(pts, (frame.shape[1], frame.shape[0]), seed=case["seed"])
    assert_fit_equal(fit, case["fit"], case["name"])


@pytest.mark.parametrize("case", [c for c in frame_cases() if c not in SMALL], ids=lambda c: c["name"])
def test_large_frames_fused_estimate(case):
    """estimate() on the 1080p (C1, C2 0-9) and 4K (C4) golden frames: batch 1
    takes the fused single launch (strip_kernel<.., kFused>, the 576-thread
    instantiation at 4K), from host numpy (strip-row ingest) and from HBM."""
    frame = make_frame(case["recipe"])
    assert sha(frame) == case["sha256"]
    for src in (frame, torch.from_numpy(frame).cuda()):
        area = eb.estimate(src, seed=case["seed"])
        if case["estimate"] is None:
            assert area == eb.FULL_FRAME, (case["name"], area)
        else:
            cx, cy, r, s = case["estimate"]
            assert isinstance(area, eb.CircularArea), (case["name"], area)
            assert abs(area.circle.cx - cx) <= PX_TOL and abs(area.circle.cy - cy) <= PX_TOL
            assert abs(area.circle.r - r) <= PX_TOL
            assert area.score == pytest.approx(s, rel=1e-12)
    eng = eb.ContentAreaEngine(frame.shape[0], frame.shape[1], 1, seed=case["seed"])
    assert eng.fused
    fit = eng.fits(eng.run(torch.from_numpy(frame).cuda()))[0]
    assert_fit_equal(fit, case["fit"], case["name"])
    assert eng.xs[0].cpu().tolist() == case["cand_x"]


def test_host_ingest_equals_device_frames():
    """numpy frames ship strip rows only; results equal the device-resident path."""
    specs = synth.bench_specs(6, 640, 480, seed=4)
    frames = np.stack([synth.render(s, 50 + k) for k, (_, s) in enumerate(specs)])
    a = eb.estimate_batch(list(frames))
    b = eb.estimate_batch(torch.from_numpy(frames).cuda())
    assert a == b
    eng = eb.ContentAreaEngine(480, 640, len(frames))
    host = torch.from_numpy(frames).pin_memory()
    rec_h = eng.run_host(host).clone()
    rec_d = eng.run(torch.from_numpy(frames).cuda()).cpu()
    assert torch.equal(rec_h, rec_d)
    assert eng.results(rec_d) == a


def test_batch_mixed_sizes_and_errors():
    f1 = synth.render(synth.bench_spec("clean", np.random.default_rng(1), 320, 240), 3)
    f2 = synth.render(synth.bench_spec("dark", np.random.default_rng(2), 640, 480), 4)
    bad = np.zeros((4, 4, 3), dtype=np.uint8)
    out = eb.estimate_batch([f1, bad, f2, f1])
    assert isinstance(out[1], eb.FrameError) and out[1].index == 1
    assert out[0] == out[3]
    cfg = eb.EcaConfig()
    for f, o in [(f1, out[0]), (f2, out[2])]:
        st, cx, cy, r, s, n = orc.estimate(f, cfg, 0)
        if st == 0:
            assert abs(o.circle.cx - cx) <= PX_TOL and abs(o.circle.r - r) <= PX_TOL
        else:
            assert o == eb.FULL_FRAME
    assert eb.estimate_batch([]) == []


def test_c2_batch_1080p_vs_oracle():
    """The bench workload (C2): 1080p mix through one fused launch vs the oracle."""
    specs = synth.bench_specs(24, 1920, 1080, seed=2024)
    frames = np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])
    eng = eb.ContentAreaEngine(1080, 1920, len(frames))
    rec = eng.run(torch.from_numpy(frames).cuda())
    got = eng.fits(rec)
    xs = eng.xs.cpu().numpy()
    cfg = eb.EcaConfig()
    for k in range(len(frames)):
        ox, oy, osc, rows, _ = orc.handcrafted_candidates(frames[k], cfg)
        assert xs[k].tolist() == ox.tolist(), k
        assert close_scores(eng.sc[k].cpu().numpy(), osc).all(), k
        keep = orc.keep_mask(ox, oy, osc, 1920, 1080, cfg)
        want = orc.ransac(ox[keep], oy[keep], osc[keep], 1920, 1080, cfg, 0)
        assert_fit_equal(got[k], want, k)


def test_pipelined_matches_run():
    """run_pipelined (bounds on the current stream, rescore + fit on a side
    stream overlapping the next batch) gives run()'s records, batch by batch."""
    specs = synth.bench_specs(40, 1920, 1080, seed=2024)
    frames = torch.from_numpy(np.stack([synth.render(s, 30000 + k)
                                        for k, (_, s) in enumerate(specs)])).cuda()
    B = 20
    eng = eb.ContentAreaEngine(1080, 1920, B)
    assert not eng.fused
    order = [0, 1, 1, 0, 1, 0, 0]
    want = {i: eng.run(frames[i * B:(i + 1) * B]).clone() for i in (0, 1)}
    got = []
    for i in order:
        rec = eng.run_pipelined(frames[i * B:(i + 1) * B])
        if len(got) % 3 == 2:
            torch.cuda.current_stream().synchronize()
        got.append((i, rec))
        if len(got) >= 2:   # a record set is reused two calls later: read it now
            eng.fence()
            j, r = got[-2]
            assert torch.equal(r, want[j]), len(got)
    eng.fence()
    j, r = got[-1]
    assert torch.equal(r, want[j])


def test_pipelined_long_stream_matches_run():
    """40 unsynchronised run_pipelined calls over 3 distinct batches (the
    buffer-set rotation with its device-side reuse guard and overlapping
    programmatic launches on reused sets): the last PIPE_SETS steps' records
    all equal run()'s."""
    specs = synth.bench_specs(40, 960, 540, seed=2024)
    frames = torch.from_numpy(np.stack([synth.render(s, 31000 + k)
                                        for k, (_, s) in enumerate(specs)])).cuda()
    B = 24
    pool = frames[[k % 40 for k in range(3 * B)]]
    eng = eb.ContentAreaEngine(540, 960, B)
    want = [eng.run(pool[k * B:(k + 1) * B]).clone() for k in range(3)]
    recs = [(i % 3, eng.run_pipelined(pool[(i % 3) * B:(i % 3 + 1) * B])) for i in range(40)]
    eng.fence()
    torch.cuda.synchronize()
    for k, r in recs[-eng.PIPE_SETS:]:
        assert torch.equal(r, want[k])


def test_pipeline_graph_replay_matches_run():
    """capture_pipelined + replay_pipelined (the bench's 1-GPU mode: a whole
    rotation of batches as one CUDA graph with both streams and the
    programmatic-dependent bounds launches as nodes) gives run()'s records for
    the last three batches (the pipeline's buffer sets), replay after replay."""
    specs = synth.bench_specs(40, 1920, 1080, seed=2024)
    frames = torch.from_numpy(np.stack([synth.render(s, 30000 + k)
                                        for k, (_, s) in enumerate(specs)])).cuda()
    B, n = 20, 5
    pool = frames[[k % 40 for k in range(n * B)]]
    eng = eb.ContentAreaEngine(1080, 1920, B)
    want = [eng.run(pool[k * B:(k + 1) * B]).clone() for k in range(n)]
    eng.run_pipelined(pool[:B])   # eager steps before capture are allowed
    eng.fence()
    eng.capture_pipelined([pool[k * B:(k + 1) * B] for k in range(n)])
    for rep in range(3):
        for rec in eng.replay_pipelined():
            rec.zero_() if rep == 1 else None
        torch.cuda.synchronize()
        recs = eng.replay_pipelined()
        torch.cuda.synchronize()
        for k in range(n - 3, n):
            assert torch.equal(recs[k], want[k]), (rep, k)


def test_split_stages_match_points():
    """eca_bounds_handcrafted + eca_rescore_handcrafted == eca_points_handcrafted."""
    import ctypes
    from paper_2210_14771_b200 import _lib, api
    specs = synth.bench_specs(12, 1280, 720, seed=5)
    frames = torch.from_numpy(np.stack([synth.render(s, 7 + k) for k, (_, s) in enumerate(specs)])).cuda()
    eng = eb.ContentAreaEngine(720, 1280, len(frames))
    eng.points(frames)
    torch.cuda.synchronize()
    ref = (eng.xs.clone(), eng.ys.clone(), eng.sc.clone())
    lib = _lib.load()
    xs, ys, sc = torch.zeros_like(ref[0]), torch.zeros_like(ref[1]), torch.zeros_like(ref[2])
    st = api._stream(eng.device)
    _lib.check(lib.eca_bounds_handcrafted(
        ctypes.c_void_p(frames.data_ptr()), len(frames), frames.stride(0), frames.stride(1), eng._rows,
        None, eng.n_strips, ctypes.byref(eng.params), api._ptr(xs), api._ptr(ys), api._ptr(sc),
        api._ptr(eng.workspace), 0, st), "bounds")
    _lib.check(lib.eca_rescore_handcrafted(
        len(frames), eng._rows, eng.n_strips, ctypes.byref(eng.params), api._ptr(xs), api._ptr(ys),
        api._ptr(sc), api._ptr(eng.workspace), st), "rescore")
    torch.cuda.synchronize()
    assert torch.equal(xs, ref[0]) and torch.equal(ys, ref[1]) and torch.equal(sc, ref[2])
    assert lib.eca_rescore_handcrafted(1, eng._rows, eng.n_strips, None, api._ptr(xs), api._ptr(ys),
                                       api._ptr(sc), api._ptr(eng.workspace), st) == _lib.ECA_ERR_ARG
    assert lib.eca_bounds_handcrafted(
        ctypes.c_void_p(frames.data_ptr()), len(frames), frames.stride(0), frames.stride(1), eng._rows,
        None, eng.n_strips, ctypes.byref(eng.params), api._ptr(xs), api._ptr(ys), api._ptr(sc),
        api._ptr(eng.workspace), 8, st) == _lib.ECA_ERR_ARG


@pytest.mark.parametrize("w,h,pad", [(333, 241, 7), (517, 300, 1), (1001, 480, 13), (2049, 200, 5),
                                     (64, 40, 3)])
def test_points_odd_sizes_and_strides(w, h, pad):
    """Odd widths and padded, unaligned row strides: the bound-and-prune
    kernel's unaligned loads, both halves' staging and the fused path against
    the oracle."""
    specs = synth.bench_specs(5, w, h, seed=w + h)
    frames = np.stack([synth.render(s, 11 + k) for k, (_, s) in enumerate(specs)])
    b = len(frames)
    rs = 3 * w + pad                        # row stride (bytes), not a multiple of 4
    fs = h * rs + 9                         # frame stride
    buf = torch.zeros(b * fs + 64, dtype=torch.uint8, device="cuda")
    t = torch.as_strided(buf[1:], (b, h, w, 3), (fs, rs, 3, 1))   # odd base address too
    t.copy_(torch.from_numpy(frames).cuda())
    cfg = eb.EcaConfig()
    want = [orc.handcrafted_candidates(frames[k], cfg) for k in range(b)]
    eng = eb.ContentAreaEngine(h, w, b)
    eng.points(t)                           # bounds + rescore (workspace path)
    xs, sc = eng.xs.cpu().numpy(), eng.sc.cpu().numpy()
    for k in range(b):
        assert xs[k].tolist() == want[k][0].tolist(), (k, xs[k], want[k][0])
        assert close_scores(sc[k], want[k][2]).all(), k
    rec = eng.run(t)                        # b <= 16: the fused single launch
    for k, fit in enumerate(eng.fits(rec)):
        ox, oy, osc = want[k][0], want[k][1], want[k][2]
        keep = orc.keep_mask(ox, oy, osc, w, h, cfg)
        assert_fit_equal(fit, orc.ransac(ox[keep], oy[keep], osc[keep], w, h, cfg, 0), k)


def test_zero_copy_host_frames_match_run():
    """ECA_BOUNDS_ZERO_COPY: the bound-and-prune kernel reads pinned host
    frames chunk by chunk over PCIe; records equal the device-resident path,
    and fewer bytes than the strip rows cross the bus."""
    specs = synth.bench_specs(20, 1920, 1080, seed=2024)
    frames = np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])
    eng = eb.ContentAreaEngine(1080, 1920, len(frames))
    want = eng.run(torch.from_numpy(frames).cuda()).clone()
    host = torch.from_numpy(frames).pin_memory()
    b0 = eng.zero_copy_bytes()
    got = eng.run_host_zero_copy(host).clone()
    assert torch.equal(got, want.cpu())
    moved = eng.zero_copy_bytes() - b0
    strip_bytes = len(frames) * eng.n_strips * 3 * 1920 * 3
    assert 0 < moved < strip_bytes
    # device frames through the same chunked loads (ECA_BOUNDS_ZERO_COPY on HBM)
    import ctypes
    from paper_2210_14771_b200 import _lib, api
    f = torch.from_numpy(frames).cuda()
    lib = _lib.load()
    _lib.check(lib.eca_bounds_handcrafted(
        ctypes.c_void_p(f.data_ptr()), len(frames), f.stride(0), f.stride(1), eng._rows, None,
        eng.n_strips, ctypes.byref(eng.params), api._ptr(eng.xs), api._ptr(eng.ys), api._ptr(eng.sc),
        api._ptr(eng.workspace), _lib.BOUNDS_ZERO_COPY, api._stream(eng.device)), "bounds")
    _lib.check(lib.eca_rescore_handcrafted(
        len(frames), eng._rows, eng.n_strips, ctypes.byref(eng.params), api._ptr(eng.xs),
        api._ptr(eng.ys), api._ptr(eng.sc), api._ptr(eng.workspace), api._stream(eng.device)), "rs")
    xs = eng.xs.clone()
    eng.points(f)
    assert torch.equal(xs, eng.xs)


def test_host_pipelined_matches_run_host():
    """run_host_pipelined (zero-copy reads, records D2H on the side stream,
    overlapping steps) lands the same records in host memory as run_host."""
    specs = synth.bench_specs(40, 1920, 1080, seed=2024)
    frames = np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])
    B = 20
    eng = eb.ContentAreaEngine(1080, 1920, B)
    hosts = [torch.from_numpy(frames[i * B:(i + 1) * B]).pin_memory() for i in (0, 1)]
    want = [eng.run_host(h).clone() for h in hosts]
    recs = [torch.zeros((B, 5), dtype=torch.float64).pin_memory() for _ in range(2)]
    for i in range(4):
        eng.run_host_pipelined(hosts[i % 2], recs[i % 2])
    eng.fence()
    torch.cuda.synchronize()
    assert torch.equal(recs[0], want[0]) and torch.equal(recs[1], want[1])
    with pytest.raises(ValueError):
        eng.run_host_pipelined(hosts[0].clone(), recs[0])   # not pinned


def test_native_api_argument_errors():
    """The C-ABI entry points added for streaming reject bad arguments."""
    import ctypes
    from paper_2210_14771_b200 import _lib, api
    lib = _lib.load()
    eng = eb.ContentAreaEngine(480, 640, 20)
    n = ctypes.c_int64()
    assert lib.eca_pipeline_bytes(0, 16, ctypes.byref(n)) == _lib.ECA_ERR_ARG
    assert lib.eca_pipeline_bytes(20, 16, ctypes.byref(n)) == _lib.ECA_OK and n.value > 0
    scratch = torch.zeros(n.value, dtype=torch.uint8, device="cuda")
    pl = ctypes.c_void_p()
    # too-small scratch, then mismatched params
    assert lib.eca_pipeline_create(20, 480, 640, eng._rows, eng.n_strips, ctypes.byref(eng.params),
                                   api._ptr(eng.trip), api._ptr(scratch), n.value - 1,
                                   ctypes.byref(pl)) == _lib.ECA_ERR_ARG
    assert lib.eca_pipeline_create(20, 480, 641, eng._rows, eng.n_strips, ctypes.byref(eng.params),
                                   api._ptr(eng.trip), api._ptr(scratch), n.value,
                                   ctypes.byref(pl)) == _lib.ECA_ERR_ARG
    assert lib.eca_pipeline_create(20, 480, 640, eng._rows, eng.n_strips, ctypes.byref(eng.params),
                                   api._ptr(eng.trip), api._ptr(scratch), n.value,
                                   ctypes.byref(pl)) == _lib.ECA_OK
    f = torch.zeros((20, 480, 640, 3), dtype=torch.uint8, device="cuda")
    out = ctypes.c_void_p()
    st = api._stream(eng.device)
    assert lib.eca_pipeline_step(pl, ctypes.c_void_p(f.data_ptr()), f.stride(0), f.stride(1), 16, None, st,
                                 ctypes.byref(out)) == _lib.ECA_ERR_ARG           # unknown flag
    assert lib.eca_pipeline_step(pl, ctypes.c_void_p(f.data_ptr()), f.stride(0), 100, 0, None, st,
                                 ctypes.byref(out)) == _lib.ECA_ERR_ARG           # row stride < 3W
    assert lib.eca_pipeline_step(pl, ctypes.c_void_p(f.data_ptr()), f.stride(0), f.stride(1), 0, None, st,
                                 ctypes.byref(out)) == _lib.ECA_OK
    assert lib.eca_pipeline_fence(pl, st) == _lib.ECA_OK
    torch.cuda.synchronize()
    rec = torch.empty((20, 5), dtype=torch.float64, device="cuda")
    rec.view(torch.uint8).view(-1).copy_(scratch[out.value - scratch.data_ptr():][:20 * 40])
    assert (eng.status(rec) == _lib.NO_CANDIDATES).all()   # black frames: no candidates
    assert lib.eca_pipeline_destroy(pl) == _lib.ECA_OK
    # the learned entry point rejects unknown flags
    net = eb.EdgeNet(eb.ChannelStats([100.0] * 3, [50.0] * 3), seed=0)
    el = eb.ContentAreaEngine(480, 640, 2, variant=eb.Learned(net))
    assert lib.eca_points_learned_ex(ctypes.c_void_p(f.data_ptr()), 2, f.stride(0), f.stride(1), el._rows,
                                     None, el.n_strips, 480, 640, api._ptr(el.w_dev), el.norm, 4,
                                     api._ptr(el.probs), api._ptr(el.xs), api._ptr(el.ys),
                                     api._ptr(el.sc), st) == _lib.ECA_ERR_ARG


def test_zero_copy_padded_host_strides():
    """Zero-copy reads from pinned host frames with padded, unaligned rows."""
    w, h, b, pad = 1001, 480, 18, 7
    specs = synth.bench_specs(b, w, h, seed=9)
    frames = np.stack([synth.render(s, 70 + k) for k, (_, s) in enumerate(specs)])
    rs = 3 * w + pad
    fs = h * rs + 5
    host = torch.zeros(b * fs + 32, dtype=torch.uint8).pin_memory()
    view = torch.as_strided(host[3:], (b, h, w, 3), (fs, rs, 3, 1))
    view.copy_(torch.from_numpy(frames))
    eng = eb.ContentAreaEngine(h, w, b)
    want = eng.run(torch.from_numpy(frames).cuda()).cpu()
    assert torch.equal(eng.run_host_zero_copy(view).clone(), want)


def test_graph_replay_matches_direct():
    frame = synth.c1_frame()
    t = torch.from_numpy(frame).cuda().unsqueeze(0)
    eng = eb.ContentAreaEngine(1080, 1920, 1)
    direct = eng.run(t).clone()
    eng.capture(t)
    for _ in range(3):
        rep = eng.replay().clone()
        assert torch.equal(rep, direct)
    assert eng.fits(direct)[0] == eb.fit_area(eb.get_points(frame), (1920, 1080))


def test_learned_matches_reference():
    npz = load_npz("learned.npz")
    net = eb.EdgeNet(eb.ChannelStats([100.0] * 3, [50.0] * 3), seed=0)
    for i in range(4):
        assert np.array_equal(net.layers[i].kernel, npz[f"w{i}"])
    assert eb.save_weights(net) == npz["blob"].tobytes()
    agree = total = 0
    for c in load_json("learned.json"):
        frame = make_frame(c["recipe"])
        rows, _ = eb.score_frame_strips(frame, eb.Learned(net))
        got = np.stack([r.scores for r in rows])
        want = npz[c["name"]]
        assert np.abs(got - want).max() <= 1e-5
        xs = [r.left_best.x for r in rows] + [r.right_best.x for r in rows]
        for k, (gx, wx) in enumerate(zip(xs, c["cand_x"])):
            total += 1
            if gx == wx:
                agree += 1
            else:   # a disagreement must be a near-tie in the reference's own scores
                row = want[k % len(rows)]
                assert abs(row[gx] - row[wx]) <= 2e-6 * max(row[wx], 1e-30), (c["name"], k)
    assert agree / total >= 0.9


def test_learned_simt_and_tensor_cores_match_reference():
    """Both CNN kernels -- tcgen05 (default, 3xTF32) and SIMT (ECA_LEARNED_SIMT)
    -- give probabilities within 1e-5 of the reference; their candidates agree
    except at near-ties."""
    npz = load_npz("learned.npz")
    net = eb.EdgeNet(eb.ChannelStats([100.0] * 3, [50.0] * 3), seed=0)
    for c in load_json("learned.json"):
        frame = make_frame(c["recipe"])
        h, w = frame.shape[:2]
        t = torch.from_numpy(frame).cuda().unsqueeze(0)
        e_tc = eb.ContentAreaEngine(h, w, 1, variant=eb.Learned(net), tensor_cores=True)
        e_ref = eb.ContentAreaEngine(h, w, 1, variant=eb.Learned(net), tensor_cores=False)
        e_tc.run(t)
        e_ref.run(t)
        torch.cuda.synchronize()
        got = e_tc.probs[0].cpu().numpy()
        want = npz[c["name"]][:, 3:w - 3]
        assert np.abs(got - want).max() <= 1e-5, c["name"]
        assert np.abs(e_ref.probs[0].cpu().numpy() - want).max() <= 1e-5, c["name"]
        assert np.abs(got - e_ref.probs[0].cpu().numpy()).max() <= 1e-5
        xt, xr = e_tc.xs[0].cpu().tolist(), e_ref.xs[0].cpu().tolist()
        full = npz[c["name"]]
        for k, (a, b) in enumerate(zip(xt, xr)):
            if a != b:
                row = full[k % len(full)]
                assert abs(row[a] - row[b]) <= 2e-5, (c["name"], k)


def test_mask_bit_exact_vs_oracle():
    rng = np.random.default_rng(0)
    circles = [eb.Circle(319.5, 239.5, 200.0), eb.Circle(10.25, 400.75, 333.3),
               eb.Circle(320.0, 240.0, 100.0), eb.Circle(-50.0, 240.0, 80.0),
               eb.Circle(319.5, 239.5, 0.5), eb.Circle(0.0, 0.0, 1e-3)]
    circles += [eb.Circle(float(rng.uniform(-100, 740)), float(rng.uniform(-100, 580)),
                          float(rng.uniform(0.1, 600))) for _ in range(40)]
    areas = [eb.CircularArea(c, 1.0) for c in circles] + [eb.FULL_FRAME]
    masks = eb.draw_mask(areas, 480, 640).cpu().numpy()
    for m, c in zip(masks, circles):
        assert np.array_equal(m, orc.disk_mask(c.cx, c.cy, c.r, 480, 640)), c
    assert masks[-1].all()
    odd = eb.draw_mask(eb.CircularArea(eb.Circle(50.3, 20.7, 17.0), 1.0), 41, 101).cpu().numpy()
    assert np.array_equal(odd, orc.disk_mask(50.3, 20.7, 17.0, 41, 101))


def test_mask_1080p_flat_path_bit_exact():
    """Packed 1080p masks take the span writer (W % 16 == 0): a batch of 9
    frames (rows of consecutive frames share a CTA's span), against the oracle."""
    circles = [eb.Circle(958.88, 545.03, 759.54), eb.Circle(959.5, 539.5, 1200.0),
               eb.Circle(0.5, 0.5, 300.25), eb.Circle(1919.0, 1079.0, 77.7), eb.Circle(960.0, -500.0, 600.0),
               eb.Circle(-10.0, 540.0, 9.0), eb.Circle(960.0, 540.0, 0.75), eb.Circle(300.1, 900.9, 410.4)]
    areas = [eb.CircularArea(c, 1.0) for c in circles] + [eb.FULL_FRAME]
    masks = eb.draw_mask(areas, 1080, 1920).cpu().numpy()
    for m, c in zip(masks, circles):
        assert np.array_equal(m, orc.disk_mask(c.cx, c.cy, c.r, 1080, 1920)), c
    assert masks[-1].all()


def test_crop_bounds_match_reference():
    fails = []
    for c in load_json("crops.json"):
        got = eb.crop_bounds([eb.Circle(*c["circle"])], c["h"], c["w"])[0]
        want = tuple(c["bounds"]) if c["bounds"] is not None else None
        if got != want:
            fails.append((c, got))
    assert not fails, fails[:3]


def test_crop_area_copies_pixels():
    frame = synth.c1_frame()
    area = eb.estimate(frame)
    crop = eb.crop_area(frame, area)
    x0, y0, x1, y1 = orc.crop_bounds(area.circle.cx, area.circle.cy, area.circle.r, 1920, 1080)
    assert np.array_equal(crop.cpu().numpy(), frame[y0:y1 + 1, x0:x1 + 1])
    with pytest.raises(ValueError):
        eb.crop_area(frame, eb.FULL_FRAME)


def test_crop_copy_packed_batch_every_alignment():
    """K5 copy through the C ABI: packed crops at every source byte offset
    (3·x0 mod 4) and every destination offset mod 16, widths below and above
    one 16-B vector, skipped (-1) entries in between."""
    from paper_2210_14771_b200 import _lib, api
    rng = np.random.default_rng(7)
    B, H, W = 96, 70, 301
    frames = rng.integers(0, 256, (B, H, W, 3), dtype=np.uint8)
    bounds = np.full((B, 4), -1, dtype=np.int32)
    for b in range(B):
        if b % 11 == 5:
            continue
        x0 = int(rng.integers(0, W - 1))
        x1 = int(min(W - 1, x0 + [0, 1, 4, 5, 6, 17, 40, 150, 300][b % 9]))
        y0 = int(rng.integers(0, H - 1))
        y1 = int(rng.integers(y0, H))
        bounds[b] = (x0, y0, x1, y1)
    sizes = [0 if r[0] < 0 else (r[2] - r[0] + 1) * (r[3] - r[1] + 1) * 3 for r in bounds]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    max_rows = int(max(r[3] - r[1] + 1 for r in bounds if r[0] >= 0))
    dev = torch.device("cuda:0")
    f = torch.from_numpy(frames).to(dev)
    bd = torch.from_numpy(bounds).to(dev)
    od = torch.from_numpy(offs).to(dev)
    out = torch.zeros(int(sum(sizes)) + 64, dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().eca_crop_copy(api._ptr(f), B, f.stride(0), f.stride(1), api._ptr(bd),
                                         api._ptr(od), api._ptr(out), max_rows, api._stream(dev)),
               "eca_crop_copy")
    got = out.cpu().numpy()
    for b, r in enumerate(bounds):
        if r[0] < 0:
            continue
        want = frames[b, r[1]:r[3] + 1, r[0]:r[2] + 1].reshape(-1)
        assert np.array_equal(got[offs[b]:offs[b] + sizes[b]], want), (b, r)
    assert not got[int(sum(sizes)):].any()


@pytest.mark.parametrize("w,h", [(40, 30), (128, 64), (134, 40), (250, 97), (517, 300), (1920, 60)])
@pytest.mark.parametrize("tc", [True, False])
def test_learned_tile_edges_match_oracle(w, h, tc):
    """CNN tiles: widths below one tile, at and around the tcgen05 tile's 122
    valid outputs, ragged last tiles; probabilities against the oracle's FP32
    network within 1e-5, batch of 3 frames."""
    rng = np.random.default_rng(w * 7 + h)
    frames = rng.integers(0, 256, (3, h, w, 3), dtype=np.uint8)
    net = eb.EdgeNet(eb.ChannelStats([90.0, 100.0, 110.0], [40.0, 50.0, 60.0]), seed=w)
    layers = [(l.kernel, l.bias) for l in net.layers]
    eng = eb.ContentAreaEngine(h, w, 3, variant=eb.Learned(net), tensor_cores=tc)
    eng.run(torch.from_numpy(frames).cuda())
    torch.cuda.synchronize()
    rows = eb.strip_heights(h, 16, 8.0)
    for k in range(3):
        want = orc.cnn_probs(orc.rgbxy_windows(frames[k], rows, [90.0, 100.0, 110.0], [40.0, 50.0, 60.0]),
                             layers)
        got = eng.probs[k].cpu().numpy()[:len(rows)]
        assert np.abs(got - want).max() <= 1e-5, (k, np.abs(got - want).max())


try:
    from hypothesis import given, settings
    from hypothesis import strategies as st
except ImportError:   # pragma: no cover
    given = None

if given is not None:
    @given(data=st.data())
    @settings(max_examples=60, deadline=None)
    def test_ransac_fuzz_matches_oracle(data):
        """Random candidate sets -- points near a random circle plus outliers,
        ragged counts, random seeds, exhaustive or seeded -- through the GPU
        fitter against the oracle: status and inlier count exact, circle within
        1e-3 px, score rel 1e-12 (fitting.py:159-230; cf. the reference's
        test_accepted_fits_always_satisfy_gates)."""
        w, h = data.draw(st.sampled_from([(640, 480), (1920, 1080), (300, 200)]))
        cx = data.draw(st.floats(0.2 * w, 0.8 * w))
        cy = data.draw(st.floats(0.2 * h, 0.8 * h))
        r = data.draw(st.floats(0.12 * w, 0.75 * w))
        n_in = data.draw(st.integers(0, 28))
        n_out = data.draw(st.integers(0, 8))
        seed = data.draw(st.integers(0, 2**31 - 1))
        rng = np.random.default_rng(seed)
        t = rng.uniform(0, 2 * np.pi, n_in)
        pts = np.column_stack([cx + r * np.cos(t) + rng.normal(0, 1.0, n_in),
                               cy + r * np.sin(t) + rng.normal(0, 1.0, n_in)])
        pts = np.vstack([pts, rng.uniform([3, 3], [w - 4, h - 4], (n_out, 2))])
        pts = np.clip(np.rint(pts), [3, 3], [w - 4, h - 4]).astype(int)
        scores = rng.uniform(0.05, 1.0, len(pts))
        cfg = eb.EcaConfig()
        exhaustive = data.draw(st.booleans()) and len(pts) <= 12
        cands = [eb.EdgeCandidate(int(x), int(y), float(s), eb.Side.LEFT) for (x, y), s in zip(pts, scores)]
        got = eb.ransac_fit(cands, (w, h), cfg, seed % 1000, exhaustive=exhaustive)
        want = orc.ransac(pts[:, 0], pts[:, 1], scores, w, h, cfg, seed % 1000, exhaustive=exhaustive)
        assert_fit_equal(got, want, (w, h, cx, cy, r, n_in, n_out, seed))


def test_run_stream_matches_run():
    """eca_pipeline_run (K steps in one native call over a pool of batches)
    gives run()'s records for the last PIPE_SETS steps."""
    specs = synth.bench_specs(40, 960, 540, seed=2024)
    frames = torch.from_numpy(np.stack([synth.render(s, 32000 + k)
                                        for k, (_, s) in enumerate(specs)])).cuda()
    B = 20
    pool = frames[[k % 40 for k in range(3 * B)]].contiguous()
    eng = eb.ContentAreaEngine(540, 960, B)
    want = [eng.run(pool[k * B:(k + 1) * B]).clone() for k in range(3)]
    recs = eng.run_stream(pool, first=1, steps=11)
    torch.cuda.synchronize()
    assert len(recs) == eng.PIPE_SETS
    for j, r in zip(range(11 - eng.PIPE_SETS, 11), recs):
        assert torch.equal(r, want[(1 + j) % 3]), j
