"""Timing of the streamed step (one launch per batch) vs its parts, 1080p C2 pool.

    python tools/time_pipe.py
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2210_14771_b200 as eb  # noqa: E402
from support import synth  # noqa: E402

B, H, W, POOL, NB = 256, 1080, 1920, 2048, 40
dev = torch.device("cuda", 0)
specs = synth.bench_specs(NB, W, H, seed=2024)
base = torch.from_numpy(np.stack([synth.render(s, 30000 + k) for k, (_, s) in enumerate(specs)])).to(dev)
pool = torch.empty((POOL, H, W, 3), dtype=torch.uint8, device=dev)
for i in range(POOL):
    pool[i].copy_(base[i % NB])
n_slots = POOL // B
eng = eb.ContentAreaEngine(H, W, B, device=dev)
st = torch.cuda.current_stream()


def timed(fn, steps, warm=5):
    for i in range(warm):
        fn(i)
    eng.fence()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record(st)
    for i in range(steps):
        fn(warm + i)
    eng.fence()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps * 1e3, (time.perf_counter() - w0) / steps * 1e6


def sl(i):
    return pool[(i % n_slots) * B:(i % n_slots + 1) * B]


want = [eng.run(sl(i)).clone() for i in range(n_slots)]
for ready in (True, False):
    recs = [(i, eng.run_pipelined(sl(i), frames_ready=ready)) for i in range(4)]
    eng.fence()
    torch.cuda.synchronize()
    assert all(torch.equal(r, want[i % n_slots]) for i, r in recs), "pipelined != run"
    for steps in (20, 200):
        r = [timed(lambda i: eng.run_pipelined(sl(i), frames_ready=ready), steps) for _ in range(3)]
        us = sorted(x[0] for x in r)
        host = sorted(x[1] for x in r)[1]
        print(f"pipelined ready={ready} steps={steps}: {us[1]:.1f} us/step (min {us[0]:.1f} max {us[2]:.1f}; host {host:.1f} us)")
torch.cuda.synchronize()
w0 = time.perf_counter()
for i in range(100):
    eng.run_pipelined(sl(i), frames_ready=True)
w1 = time.perf_counter()
eng.fence()
torch.cuda.synchronize()
print(f"host enqueue only: {(w1 - w0) / 100 * 1e6:.1f} us/step")
us, _ = timed(lambda i: eng.run(sl(i)), 100)
print(f"run() single launch, no overlap: {us:.1f} us")
us, _ = timed(lambda i: eng.bounds(sl(i), overlap=True, slot=i % 4), 100)
print(f"bounds only, overlapped: {us:.1f} us")
us, _ = timed(lambda i: eng.bounds(sl(i), overlap=False, slot=i % 4), 100)
print(f"bounds only, isolated: {us:.1f} us")
# graph of a whole rotation
eng.capture_pipelined([sl(i) for i in range(n_slots)])
us, _ = timed(lambda i: eng.replay_pipelined(), 20)
print(f"graph replay of {n_slots} steps: {us / n_slots:.1f} us/step")
# latency: batch 1, fused strip kernel vs single-launch final-stage kernel
frame = torch.from_numpy(synth.c1_frame()).to(dev).unsqueeze(0)
for name, e in (("fused strip", eb.ContentAreaEngine(H, W, 1, device=dev)),):
    e.capture(frame)
    ts = []
    for _ in range(300):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        e.replay()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"latency {name}: p50 {np.percentile(ts, 50):.1f} us")
e = eb.ContentAreaEngine(H, W, 1, device=dev)
e.fused = False
e.capture(frame)
ts = []
for _ in range(300):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    e.replay()
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print(f"latency final-stage kernel B=1: p50 {np.percentile(ts, 50):.1f} us")
assert torch.equal(e.rec, eb.ContentAreaEngine(H, W, 1, device=dev).run(frame))
# native K-step call (bench path), 20 steps, after an idle pause vs warm
for pause in (0.0, 0.2):
    r = []
    for rep in range(3):
        eng.run_stream(pool, 0, 5)
        eng.fence()
        torch.cuda.synchronize()
        time.sleep(pause)
        if pause:
            eng.run_stream(pool, 0, 5) if rep == 2 else None   # rep 2: warm-up right before
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.run_stream(pool, 5, 20)
        eng.fence()
        b.record(st)
        torch.cuda.synchronize()
        r.append(a.elapsed_time(b) / 20 * 1e3)
    print(f"run_stream 20 steps, pause {pause}: " + ", ".join(f"{x:.1f}" for x in r) + " us/step")
