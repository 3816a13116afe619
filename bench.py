"""Benchmark of the content-area hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = the handcrafted pipeline (estimate: strip scoring -> candidates ->
filter -> seeded RANSAC) over one batch of 256 synthetic 1080p frames
(config C2); for N > 1 (torchrun, one process per GPU) every
rank runs its own batch and the 40-byte per-frame records are all-gathered
with NCCL.  Steps stream: the FP64 rescore + fit of batch i run on a side
stream under the bound-and-prune kernel of batch i+1 (ContentAreaEngine.
run_pipelined); the timed region ends after the last batch's fit.  Rank 0
prints ONE JSON line.

value : frames/s, whole job, frames already resident in HBM (a 2048-slot pool,
        566 MB of strip rows, so every step reads DRAM, not L2)
e2e   : frames/s from pinned HOST frames to host records through
        ContentAreaEngine.run_host_pipelined: the kernel reads the strip rows it
        visits over PCIe (zero-copy TMA), records D2H every step, steps overlap
        (synchronous and H2D-copy paths reported beside it)
--impl reference : the reference algorithm on the host cores (the numpy
        oracle port of /root/reference's eca package; the reference itself is
        pure Python and cannot be shipped to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BATCH, HEIGHT, WIDTH = 256, 1080, 1920
POOL = 2048
N_BASE = 40
METRIC = "1080p frames/sec & p50 ms/frame at 1/2/4/8 B200; % HBM roofline vs CPU ref"
UNIT = "frames/s"
# algorithmic bytes per frame of the dominant kernel:
# 16 strips x 3 rows (h-1, h, h+1) x 1920 px x 3 B read
STRIP_BYTES_PER_FRAME = 16 * 3 * WIDTH * 3
WORKLOAD = ("C2: handcrafted estimate (strip scoring + candidates + filter + seeded RANSAC/LSQ) "
            "on 256 synthetic 1080p RGB frames, benchmark_specs(seed=2024) 5-category mix")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ frames ---
def _render(k: int) -> np.ndarray:
    from support import synth
    specs = synth.bench_specs(k + 1, WIDTH, HEIGHT, seed=2024)
    return synth.render(specs[k][1], 30000 + k)


def base_frames(n: int = N_BASE) -> np.ndarray:
    workers = max(1, min(n, (os.cpu_count() or 1)))
    with ProcessPoolExecutor(workers) as ex:
        frames = list(ex.map(_render, range(n)))
    return np.stack(frames)


# ------------------------------------------------------------------ clocks ---
class ClockSampler:
    """SM clock + throttle reasons while the timed region runs, sampled by an
    `nvidia-smi -lms` subprocess (off the interpreter that enqueues the steps)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int, period_ms: int = 20):
        self.index, self.period = index, period_ms
        self.proc, self.max_mhz = None, None
        self.samples, self.reasons = [], set()

    def __enter__(self):
        import shutil
        import subprocess
        smi = shutil.which("nvidia-smi")
        if smi:
            try:
                self.max_mhz = int(subprocess.run(
                    [smi, "-i", str(self.index), "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=20).stdout.strip() or 0) or None
                self.proc = subprocess.Popen(
                    [smi, "-i", str(self.index), "--query-gpu=clocks.sm,clocks_event_reasons.active",
                     "--format=csv,noheader,nounits", "-lms", str(self.period)],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                time.sleep(0.2)   # first sample before the timed region starts
            except Exception as exc:  # noqa: BLE001
                log("clock sampling unavailable:", exc)
                self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            return
        time.sleep(2.5 * self.period / 1000)   # a sample after the region
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=20)
        for line in out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 2:
                continue
            try:
                self.samples.append(int(parts[0]))
                bits = int(parts[1], 16)
            except ValueError:
                continue
            for bit, name in self.REASONS.items():
                if bits & bit:
                    self.reasons.add(name)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "method": f"nvidia-smi -lms {self.period} subprocess, from just before to just after "
                          "the timed region"}


# ------------------------------------------------------------- CPU baseline ---
_CPU_FRAMES = None


def _cpu_estimate(idx: int):
    from oracle import eca_oracle as orc
    from paper_2210_14771_b200.params import EcaConfig
    return orc.estimate(_CPU_FRAMES[idx % len(_CPU_FRAMES)], EcaConfig(), 0)[0]


def cpu_pool(frames: np.ndarray):
    global _CPU_FRAMES
    _CPU_FRAMES = frames            # inherited by the forked workers
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    import multiprocessing as mp
    ex = ProcessPoolExecutor(cores, mp_context=mp.get_context("fork"))
    list(ex.map(_cpu_estimate, range(cores * 2)))   # warm the workers
    return ex, cores


def cpu_rate(ex, cores: int, n_frames: int) -> float:
    t0 = time.perf_counter()
    list(ex.map(_cpu_estimate, range(n_frames), chunksize=max(1, n_frames // (cores * 4))))
    return n_frames / (time.perf_counter() - t0)


# ---------------------------------------------------------------- reference ---
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    frames = base_frames()
    ex, cores = cpu_pool(frames)
    probe = cpu_rate(ex, cores, cores * 4)
    # per-step sample sized so warmup + steps finish in ~60 s
    per_step = int(max(cores, min(BATCH, 60.0 * probe / max(1, args.steps + args.warmup))))
    for _ in range(args.warmup):
        cpu_rate(ex, cores, per_step)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        list(ex.map(_cpu_estimate, range(per_step), chunksize=max(1, per_step // (cores * 4))))
    dt = time.perf_counter() - t0
    ex.shutdown()
    value = args.steps * per_step / dt
    sample = (f"{per_step} frames/step of the C2 1080p mix ({N_BASE} distinct renders cycled), "
              f"numpy oracle port of the reference, process pool of {cores}, 1 BLAS thread each")
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "batch": per_step, "height": HEIGHT, "width": WIDTH,
                   "parallelism": "host process pool"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------- ours ---
C5_FRAMES, C5_POOL = 100_000, 1024


def pool_base_index(i: int, rank: int) -> int:
    """Render (of the N_BASE distinct ones) in pool slot i of this rank."""
    return (i + rank * 7) % N_BASE


def oracle_records(base: np.ndarray) -> list:
    """The reference's estimate of every distinct render (numpy oracle port),
    the parity check of the timed runs' records."""
    from oracle import eca_oracle as orc
    from paper_2210_14771_b200.params import EcaConfig
    cfg = EcaConfig()
    return [orc.estimate(f, cfg, 0) for f in base]


def check_records(recs, base_idx, want) -> dict:
    """recs: (B,5) device record tensors; base_idx[k][i]: render of row i of
    recs[k]; want: oracle tuples per render.  Status / inliers exact, circle
    within 1e-3 px."""
    n = bad = 0
    for rec, idx in zip(recs, base_idx):
        for row, k in zip(_records_np(rec), idx):
            st, cx, cy, r, score, inl = want[k]
            ok = row[5] == st and (st != 0 or (abs(row[0] - cx) <= 1e-3 and abs(row[1] - cy) <= 1e-3 and
                                               abs(row[2] - r) <= 1e-3 and row[4] == inl))
            n += 1
            bad += not ok
    return {"frames_checked": n, "mismatches": bad, "distinct_renders": len(set(i for ix in base_idx for i in ix)),
            "bar": "status + inliers exact, cx/cy/r within 1e-3 px of the numpy oracle port"}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2210_14771_b200 as eb
    from paper_2210_14771_b200.engine import ContentAreaEngine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}")
    # (ECA_DIST_BACKEND=gloo: a functional dry run of the N > 1 path with every
    # rank on the box's GPUs round-robin; the measured runs use NCCL, one GPU per rank)
    backend = os.environ.get("ECA_DIST_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    base = base_frames()
    want = oracle_records(base) if rank == 0 else None
    pool = torch.empty((POOL, HEIGHT, WIDTH, 3), dtype=torch.uint8, device=dev)
    base_dev = torch.from_numpy(base).to(dev)
    for i in range(POOL):   # distinct addresses: a step never re-reads L2-resident rows
        pool[i].copy_(base_dev[pool_base_index(i, rank)])
    del base_dev
    torch.cuda.synchronize()

    eng = ContentAreaEngine(HEIGHT, WIDTH, BATCH, device=dev)
    n_slots = POOL // BATCH
    stream = torch.cuda.current_stream(dev)

    # streaming throughput mode, host-light: the K steps are ONE native call
    # (eca_pipeline_run): per batch a bound-and-prune launch + a fit launch,
    # programmatic dependent launches so batches overlap.  The pool was
    # filled before, so the kernels need not wait on the previous kernel.
    eng.run_stream(pool, 0, args.warmup)   # engine, pipeline and code paths warm
    eng.fence()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clocks:
        # the W warm-up steps again right before the timed region: the sampler's
        # start-up pause leaves the GPU idle, and the first launches after an
        # idle period run slow
        eng.run_stream(pool, 0, args.warmup)
        eng.fence()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0.record(stream)
        recs = eng.run_stream(pool, args.warmup, args.steps)
        eng.fence(stream)   # the last step's fits are inside the timed region
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = t0.elapsed_time(t1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = world * BATCH * args.steps / (ms / 1e3)
    ms_step = ms / args.steps
    parity = None
    if rank == 0:   # the timed run's last batches against the oracle (outside the timed region)
        steps_done = [args.warmup + j for j in range(args.steps - len(recs), args.steps)]
        idx = [[pool_base_index((st % n_slots) * BATCH + f, rank) for f in range(BATCH)] for st in steps_done]
        parity = check_records(recs, idx, want)

    # kernel-only timing of the step's dominant kernel (K1 bound-and-prune,
    # bounds_kernel) over the same pool, on the same stream, in two launch
    # modes: (a) as the streaming pipeline launches it -- back to back with
    # programmatic dependent launch, so a launch's first CTAs start in the
    # previous launch's tail, on 4 rotating workspaces (the roofline number);
    # (b) isolated, each launch waiting for the previous one to finish
    kt0, kt1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k_steps = max(args.steps, 50)

    def time_bounds(overlap: bool) -> float:
        for i in range(4):
            eng.bounds(pool[(i % n_slots) * BATCH:(i % n_slots + 1) * BATCH], overlap=overlap, slot=i % 4)
        torch.cuda.synchronize()
        kt0.record(stream)
        for i in range(k_steps):
            eng.bounds(pool[(i % n_slots) * BATCH:(i % n_slots + 1) * BATCH], overlap=overlap, slot=i % 4)
        kt1.record(stream)
        torch.cuda.synchronize()
        return kt0.elapsed_time(kt1) / k_steps
    k_ms = time_bounds(True)
    k_ms_isolated = time_bounds(False)
    bytes_launch = STRIP_BYTES_PER_FRAME * BATCH
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = bytes_launch / (k_ms / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")

    c5 = c5_leg(eb, dev, base, rank, world)

    # end to end through the public engine API from pinned HOST frames, 4
    # distinct host batches rotating: every step the bound-and-prune kernel
    # reads the strip rows it visits over PCIe (zero-copy TMA, bytes counted by
    # the kernel) and the fit kernel writes the records into pinned host
    # memory; steps overlap, wall clock until the last records are on the host
    hosts = [torch.from_numpy(np.stack([base[(i + 5 * h + rank) % N_BASE] for i in range(BATCH)])).pin_memory()
             for h in range(4)]
    e_steps = max(8, min(args.steps, 64))
    host_recs = [torch.zeros((BATCH, 5), dtype=torch.float64).pin_memory() for _ in range(4)]
    for i in range(max(4, args.warmup)):
        eng.run_host_pipelined(hosts[i % 4], host_recs[i % 4])
    eng.fence()
    torch.cuda.synchronize()
    b0 = eng.pipeline_zero_copy_bytes()
    if world > 1:
        dist.barrier()
    w0 = time.perf_counter()
    for i in range(e_steps):
        eng.run_host_pipelined(hosts[i % 4], host_recs[i % 4])
    eng.fence()
    torch.cuda.synchronize()
    e_wall = time.perf_counter() - w0
    h2d = (eng.pipeline_zero_copy_bytes() - b0) // e_steps
    e_ms_t = torch.tensor([e_wall * 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_ms_t, op=dist.ReduceOp.MAX)
    e2e = world * BATCH * e_steps / (float(e_ms_t.item()) / 1e3)
    e2e_parity = None
    if rank == 0:   # the last 4 host batches' records, straight from pinned memory
        idx = [[(i + 5 * ((e_steps - 4 + j) % 4) + rank) % N_BASE for i in range(BATCH)] for j in range(4)]
        e2e_parity = check_records([host_recs[(e_steps - 4 + j) % 4] for j in range(4)], idx, want)
    e2e_sync = None
    if rank == 0:   # the synchronous form (one call, host sync every step)
        for _ in range(3):
            eng.run_host_zero_copy(hosts[0])
        w0 = time.perf_counter()
        for i in range(16):
            eng.run_host_zero_copy(hosts[i % 4])
        e2e_sync = BATCH * 16 / (time.perf_counter() - w0)
    d2h = BATCH * 40

    lat = learned = mask = crop = uhd = evaluation = training = labelling = None
    if rank == 0:
        lat = latency(eb, dev)
        learned = learned_leg(eb, dev, pool, n_slots, peaks, base)
        mask = mask_leg(eb, dev, eng, pool, peaks)
        crop = crop_leg(eb, dev, eng, pool, peaks)
        uhd = uhd_leg(eb, dev, peaks)
        evaluation = eval_leg(eb, dev, eng, pool)
        training = train_leg(eb, dev)
        labelling = label_leg(eb, dev, base)
        if world == 1 and not args.no_cpu:
            learned["cpu_baseline"] = learned_cpu(base)
            evaluation["cpu_baseline"] = eval_cpu(evaluation.pop("_pairs"))
            training["cpu_baseline"] = train_cpu()
            labelling["cpu_baseline"] = label_cpu(labelling.pop("_dir"))
        evaluation.pop("_pairs", None)
        labelling.pop("_dir", None)

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            ex, cores = cpu_pool(base)
            n = int(max(cores * 8, min(2048, 20.0 * cpu_rate(ex, cores, cores * 4))))
            rate = cpu_rate(ex, cores, n)
            ex.shutdown()
            cpu = {"value": round(rate, 3), "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"{n} frames of the C2 1080p mix, numpy oracle port of the reference, "
                             f"process pool of {cores}, 1 BLAS thread each"}
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "batch_per_gpu": BATCH, "height": HEIGHT, "width": WIDTH,
                       "pool_frames": POOL, "distinct_renders": N_BASE,
                       "l2": f"inputs larger than L2: {POOL}-slot HBM pool rotated "
                             f"({POOL * STRIP_BYTES_PER_FRAME / 1e6:.0f} MB of strip rows > 126 MB L2)",
                       "parallelism": f"dp{world}: each rank streams its own batches (weak scaling); "
                                      "the 100k-frame sharded stream with NCCL record gathers is c5_stream",
                       "pipelining": "one native call enqueues the K steps (eca_pipeline_run); per step a "
                                     "bound-and-prune launch and a fit launch (FP64 rescore + RANSAC), both "
                                     "programmatic dependent launches, 4 rotating buffer sets with a "
                                     "device-side reuse guard"},
            "parity": parity,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "eca::bounds_kernel<1, 0> (K1 strip scoring: exact integer Sobel / "
                                   "preceding max, FP32 bound-and-prune, survivor slots)",
                         "kernel_share_of_step": round(k_ms / ms_step, 3),
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "kernel_ms": round(k_ms, 5),
                         "launch_mode": "as the streaming pipeline launches it: back to back with programmatic "
                                        "dependent launch (a launch's CTAs start in the previous launch's tail), "
                                        "4 rotating workspaces; kernel_ms = event time / launches",
                         "kernel_ms_isolated": round(k_ms_isolated, 5),
                         "frac_isolated": round(bytes_launch / (k_ms_isolated / 1e3) / 1e9 / peak, 4),
                         "step_frac": round(bytes_launch / (ms_step / 1e3) / 1e9 / peak, 4),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"},
            "e2e": {"value": round(e2e, 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": d2h, "steps": e_steps, "host_batches": 4, "parity": e2e_parity,
                    "path": "ContentAreaEngine.run_host_pipelined over 4 distinct pinned host batches: "
                            "every step the bound-and-prune kernel reads the strip rows it visits from "
                            "pinned host memory over PCIe (zero-copy TMA, h2d bytes counted by the kernel), "
                            "the fit kernel writes the 40-B records into pinned host memory; steps overlap, "
                            "wall clock until the last step's records are on the host",
                    "synchronous_path": None if e2e_sync is None else {
                        "value": round(e2e_sync, 2),
                        "path": "run_host_zero_copy: same reads, host sync every step"}},
            "c5_stream": c5,
            "latency_ms": lat,
            "learned": learned,
            "mask": mask,
            "crop": crop,
            "uhd_4k": uhd,
            "evaluation": evaluation,
            "training": training,
            "pseudo_labelling": labelling,
            "clocks": clocks.summary(),
            "gpu_launches": args.steps * eng.launches_per_step + 1,
            "cpu_baseline": cpu,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


def c5_leg(eb, dev, base, rank: int, world: int) -> dict:
    """BASELINE config 5: the 100k-frame 1080p stream (frame k = render of pool
    slot k mod 1024), contiguous shards per rank (ShardedEstimator): batches of
    256 through the pipeline, records written by the fit kernel into the send
    buffer, one NCCL all_gather_into_tensor per 32 batches on a side stream.
    frames/s = 100k / the slowest rank's device time."""
    import torch
    import torch.distributed as dist
    from paper_2210_14771_b200.shard import ShardedEstimator
    pool = torch.empty((C5_POOL, HEIGHT, WIDTH, 3), dtype=torch.uint8, device=dev)
    bd = torch.from_numpy(base).to(dev)
    for i in range(C5_POOL):
        pool[i].copy_(bd[i % N_BASE])
    del bd
    se = ShardedEstimator(C5_FRAMES, HEIGHT, WIDTH, device=dev, chunk=BATCH, gather_every=32)

    def frames(a, b):   # local rows [a, b) -> pool views (a batch never wraps the pool: 1024 % 256 == 0)
        k = (se.start + a) % C5_POOL
        if k + (b - a) <= C5_POOL:
            return pool[k:k + (b - a)]
        return torch.cat([pool[k:], pool[:(k + b - a) - C5_POOL]])
    torch.cuda.synchronize()
    se.run(frames, frames_ready=True)   # warm-up (engines, pipeline, NCCL)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    table = se.run(frames, frames_ready=True)
    b.record(stream)
    torch.cuda.synchronize()
    ms_t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
    per_rank = [float(ms_t.item())]
    if world > 1:
        parts = [torch.empty_like(ms_t) for _ in range(world)]
        dist.all_gather(parts, ms_t)
        per_rank = [float(p.item()) for p in parts]
    ms = max(per_rank)
    st = table.view(torch.int32).view(C5_FRAMES, 10)[:, 9]
    del pool
    torch.cuda.empty_cache()
    return {"metric": "100k-frame 1080p stream frames/s (C5: contiguous shards, NCCL gather of 40-B records)",
            "value": round(C5_FRAMES / (ms / 1e3), 1), "unit": "frames/s", "frames": C5_FRAMES,
            "ms": round(ms, 3), "rank_ms": [round(v, 3) for v in per_rank], "scaling": "strong",
            "gathers_per_rank": se.gathers, "record_bytes_gathered": C5_FRAMES * 40,
            "accepted": int((st == 0).sum().item()),
            "path": "ShardedEstimator.run: full + tail engines, run_pipelined per 256-frame batch, "
                    "all_gather_into_tensor per 32 batches on a side stream; device time on the compute "
                    "stream incl. the final gather, max over ranks"}


# FLOPs of the strip CNN per frame: 16 strips x
# 2 x [5*8*9*5*(W-2) + 8*16*9*3*(W-4) + 16*32*9*(W-6) + 32*(W-6)]
CNN_FLOP_PER_FRAME = 16 * 2 * (5 * 8 * 9 * 5 * (WIDTH - 2) + 8 * 16 * 9 * 3 * (WIDTH - 4)
                               + 16 * 32 * 9 * (WIDTH - 6) + 32 * (WIDTH - 6))


def learned_leg(eb, dev, pool, n_slots, peaks, base=None) -> dict:
    """C3: the learned variant (EdgeNet strip CNN, random-init FP32 weights
    of the reference architecture, edgenet.py) over the same 256-frame
    batches: CNN + half-row selection + fit, frames resident in HBM."""
    import torch
    from paper_2210_14771_b200.engine import ContentAreaEngine
    net = eb.EdgeNet(eb.ChannelStats([100.0] * 3, [50.0] * 3), seed=0)
    stream = torch.cuda.current_stream(dev)
    steps = 20

    def step_ms(eng):
        for i in range(3):
            eng.run(pool[(i % n_slots) * BATCH:(i % n_slots + 1) * BATCH])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for i in range(steps):
            eng.run(pool[(i % n_slots) * BATCH:(i % n_slots + 1) * BATCH])
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    eng = ContentAreaEngine(HEIGHT, WIDTH, BATCH, variant=eb.Learned(net), device=dev)
    ms = step_ms(eng)
    ms_simt = step_ms(ContentAreaEngine(HEIGHT, WIDTH, BATCH, variant=eb.Learned(net), device=dev,
                                        tensor_cores=False))
    tflops = CNN_FLOP_PER_FRAME * BATCH / (ms * 1e-3) / 1e12
    peak = peaks.get("bf16_tflops", 2250.0)
    return {"metric": "learned-variant frames/s (C3: EdgeNet strip CNN + select + fit)",
            "value": round(BATCH / (ms * 1e-3), 1), "unit": "frames/s", "ms_per_step": round(ms, 4),
            "steps": steps, "dtype": "f32 (3xTF32 on tcgen05)", "launches_per_step": eng.launches_per_run,
            "roofline": {"bound": "tensor", "achieved": round(tflops, 2), "peak": peak,
                         "unit": "TFLOP/s", "frac": round(tflops / peak, 4),
                         "kernel": "cnn_kernel_tc: the three 3x3 layers as tcgen05 kind::tf32 MMA chains "
                                   "(3xTF32), no im2col; algorithmic FP32 FLOPs (not the 3x split) over the "
                                   "step time incl. select + fit",
                         "algorithmic_flop_per_frame": CNN_FLOP_PER_FRAME,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (measured)"},
            "simt_variant": {"value": round(BATCH / (ms_simt * 1e-3), 1), "unit": "frames/s",
                             "ms_per_step": round(ms_simt, 4),
                             "kernel": "cnn_kernel: FP32 FMA on the CUDA cores (ECA_LEARNED_SIMT)"},
            "candidate_agreement": None if base is None else learned_agreement(eb, dev, net, base)}


_CPU_LCANDS = None


def _cpu_learned_cands(idx: int):
    from oracle import eca_oracle as orc
    from paper_2210_14771_b200.params import EcaConfig
    frames, layers = _CPU_LCANDS
    f = frames[idx]
    cfg = EcaConfig()
    rows = orc.strip_rows(f.shape[0], cfg.strip_count, cfg.strip_weighting)
    sc = orc.learned_scores(f, rows, [100.0] * 3, [50.0] * 3, layers)
    xs, _, _ = orc.candidates_from_scores(sc, rows)
    return xs, sc


def learned_agreement(eb, dev, net, base, n: int = 16) -> dict:
    """SURVEY 8(c) learned contract: the learned variant's half-row winners
    (3xTF32 tcgen05 CNN) against the numpy FP32 oracle on the same frames;
    every disagreement must be a near-tie in the oracle's own probabilities."""
    import torch
    from paper_2210_14771_b200.engine import ContentAreaEngine
    global _CPU_LCANDS
    from oracle import eca_oracle as orc
    frames = base[:n]
    eng = ContentAreaEngine(HEIGHT, WIDTH, n, variant=eb.Learned(net), device=dev)
    eng.run(torch.from_numpy(frames).to(dev))
    got = eng.xs.cpu().numpy()
    _CPU_LCANDS = (frames, orc.glorot_layers(0))
    import multiprocessing as mp
    with ProcessPoolExecutor(min(n, os.cpu_count() or 1), mp_context=mp.get_context("fork")) as ex:
        ref = list(ex.map(_cpu_learned_cands, range(n)))
    s = eng.n_strips
    total = agree = ties = 0
    worst = 0.0
    for k, (xs, sc) in enumerate(ref):
        for j in range(2 * s):
            total += 1
            if got[k, j] == xs[j]:
                agree += 1
                continue
            row = sc[j % s]
            gap = abs(float(row[xs[j]]) - float(row[got[k, j]]))
            worst = max(worst, gap)
            ties += gap <= 1e-5
    return {"half_rows": total, "agree": agree, "rate": round(agree / total, 6),
            "disagreements_near_tie": ties, "max_prob_gap_at_disagreement": worst,
            "frames": n, "reference": "numpy FP32 oracle port of edgenet.score_strips_learned",
            "near_tie_bar": "oracle probability gap between the two columns <= 1e-5"}


def mask_leg(eb, dev, eng, pool, peaks) -> dict:
    """draw_mask (K4) for the 256 records of one step: H*W bytes written per
    frame, event-timed; HBM-write bound."""
    import ctypes
    import torch
    from paper_2210_14771_b200 import _lib, api
    rec = eng.run(pool[:BATCH]).clone()
    out = torch.empty((BATCH, HEIGHT, WIDTH), dtype=torch.uint8, device=dev)
    lib = _lib.load()
    st = api._stream(dev)

    def launch():
        _lib.check(lib.eca_draw_mask(api._ptr(rec), BATCH, HEIGHT, WIDTH, api._ptr(out), HEIGHT * WIDTH, st),
                   "eca_draw_mask")
    for _ in range(3):
        launch()
    steps = 20
    stream = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(steps):
        launch()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    nbytes = BATCH * HEIGHT * WIDTH
    gbs = nbytes / (ms * 1e-3) / 1e9
    # a write-only kernel's ceiling: the same buffer filled with 16-byte-wide
    # int32 stores by torch, measured here (the copy peak counts reads too)
    o32 = out.view(torch.int32)
    for _ in range(3):
        o32.fill_(7)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(steps):
        o32.fill_(7)
    b.record(stream)
    torch.cuda.synchronize()
    fill_gbs = nbytes / (a.elapsed_time(b) / steps * 1e-3) / 1e9
    copy_peak = peaks.get("hbm_gbs", 6650.0)
    peak = max(copy_peak, fill_gbs)
    accepted = int((eng.status(rec) == 0).sum().item())
    return {"metric": "draw_mask masks/s (K4, 1080p uint8 masks from one step's records)",
            "value": round(BATCH / (ms * 1e-3), 1), "unit": "masks/s", "ms_per_launch": round(ms, 5),
            "accepted_circles": accepted, "frames": BATCH,
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": round(peak, 1), "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "kernel": "mask_kernel_flat (packed masks: one span "
                         "of 16-byte stores per 32 rows)",
                         "algorithmic_bytes_per_launch": nbytes,
                         "frac_of_copy_peak": round(gbs / copy_peak, 4),
                         "write_fill_gbs": round(fill_gbs, 1),
                         "peak_source": "max(MEASURED_PEAKS.json hbm_gbs (copy: read+write), a torch int32 "
                                        "fill_ of the same buffer measured in this run (write only))"}}


_CPU_LEARNED = None


def _cpu_learned(idx: int):
    from oracle import eca_oracle as orc
    from paper_2210_14771_b200.params import EcaConfig
    frames, layers = _CPU_LEARNED
    return orc.estimate(frames[idx % len(frames)], EcaConfig(), 0, layers=layers,
                        norm=([100.0] * 3, [50.0] * 3))[0]


def learned_cpu(frames) -> dict:
    """The learned variant on the host cores: the numpy oracle port of the
    reference's EdgeNet path, a process pool, a bounded sample."""
    global _CPU_LEARNED
    from oracle import eca_oracle as orc
    _CPU_LEARNED = (frames, orc.glorot_layers(0))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    import multiprocessing as mp
    with ProcessPoolExecutor(cores, mp_context=mp.get_context("fork")) as ex:
        list(ex.map(_cpu_learned, range(cores)))
        n = cores * 2
        t0 = time.perf_counter()
        list(ex.map(_cpu_learned, range(n)))
        dt = time.perf_counter() - t0
    return {"value": round(n / dt, 2), "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": f"{n} frames of the C2 1080p mix, learned variant (EdgeNet, seed 0) through the "
                      f"numpy oracle port, process pool of {cores}"}


def crop_leg(eb, dev, eng, pool, peaks) -> dict:
    """crop_augment geometry + copy (K5) for one step's records: bounds kernel,
    then the packed HWC crops (read + write bytes)."""
    import torch
    from paper_2210_14771_b200 import _lib, api
    rec = eng.run(pool[:BATCH]).clone()
    f = pool[:BATCH]
    lib = _lib.load()
    st = api._stream(dev)
    bounds = torch.empty((BATCH, 4), dtype=torch.int32, device=dev)
    _lib.check(lib.eca_crop_bounds(api._ptr(rec), BATCH, HEIGHT, WIDTH, api._ptr(bounds), st), "crop_bounds")
    bh = bounds.cpu().numpy()
    sizes = [(0 if r[0] < 0 else (r[2] - r[0] + 1) * (r[3] - r[1] + 1) * 3) for r in bh]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    offs_d = torch.from_numpy(offs).to(dev)
    out = torch.empty(max(1, int(sum(sizes))), dtype=torch.uint8, device=dev)
    max_rows = int(max([1] + [r[3] - r[1] + 1 for r in bh if r[0] >= 0]))

    def launch():
        _lib.check(lib.eca_crop_bounds(api._ptr(rec), BATCH, HEIGHT, WIDTH, api._ptr(bounds), st), "crop_bounds")
        _lib.check(lib.eca_crop_copy(api._ptr(f), BATCH, f.stride(0), f.stride(1), api._ptr(bounds),
                                     api._ptr(offs_d), api._ptr(out), max_rows, st), "crop_copy")
    for _ in range(3):
        launch()
    steps = 20
    stream = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(steps):
        launch()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    nbytes = 2 * int(sum(sizes))
    gbs = nbytes / (ms * 1e-3) / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    return {"metric": "crop_augment crops/s (K5: bounds + packed HWC copy, 1080p)",
            "value": round(BATCH / (ms * 1e-3), 1), "unit": "crops/s", "ms_per_step": round(ms, 5),
            "crops": int(sum(1 for r in bh if r[0] >= 0)),
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "kernel": "crop_bounds_kernel + crop_copy_kernel",
                         "algorithmic_bytes_per_step": nbytes}}


def eval_leg(eb, dev, eng, pool) -> dict:
    """§8f-3: normalised Hausdorff of one step's fitted records against the
    renderer's truth circles (area_errors), event-timed over the kernels of
    eca_area_hausdorff (boundary sampling + FP32-ordered exact FP64 scan)."""
    import ctypes
    import torch
    from paper_2210_14771_b200 import _lib, api, metrics
    from support import synth
    rec = eng.run(pool[:BATCH]).clone()
    specs = synth.bench_specs(N_BASE, WIDTH, HEIGHT, seed=2024)
    truth = [specs[i % N_BASE][1].circle for i in range(BATCH)]
    rt = api._area_records([t for t in truth], dev)
    dims = torch.tensor([[WIDTH, HEIGHT]] * BATCH, dtype=torch.int32, device=dev)
    lib = _lib.load()
    nb = ctypes.c_int64()
    _lib.check(lib.eca_nh_workspace_bytes(BATCH, WIDTH, HEIGHT, 1.0, ctypes.byref(nb)), "nh ws")
    ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
    hd = torch.empty(BATCH, dtype=torch.float64, device=dev)
    stt = torch.empty(BATCH, dtype=torch.int32, device=dev)
    st = api._stream(dev)

    def launch():
        _lib.check(lib.eca_area_hausdorff(api._ptr(rec), api._ptr(rt), api._ptr(dims), BATCH, WIDTH, HEIGHT,
                                          1.0, api._ptr(ws), nb.value, api._ptr(hd), api._ptr(stt), st),
                   "eca_area_hausdorff")
    for _ in range(3):
        launch()
    steps = 10
    stream = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(steps):
        launch()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    nh = hd.cpu().numpy() * (metrics.REF_DIAGONAL / math.hypot(WIDTH, HEIGHT))
    fits = [None if r[5] != 0 else (float(r[0]), float(r[1]), float(r[2]))
            for r in _records_np(rec)]
    pairs = [(f, None if t is None else (t.cx, t.cy, t.r)) for f, t in zip(fits, truth)]
    return {"metric": "normalised-Hausdorff evaluations/s (§8f-3: boundary sampling + exact Hausdorff, "
                      "1080p, fitted records vs renderer truth)",
            "value": round(BATCH / (ms * 1e-3), 1), "unit": "samples/s", "ms_per_step": round(ms, 5),
            "samples": BATCH, "launches_per_step": 6,
            "avg_error_px": round(float(nh.mean()), 4),
            "miss_pct": round(100.0 * float((nh > metrics.HIT_MAX_NH_PX).mean()), 2),
            "_pairs": pairs}


LABEL_FRAMES = 256


def label_leg(eb, dev, base) -> dict:
    """§8f-1: pseudo_label over a directory of 256 1080p PNG frames (the C2
    renders): worker processes decode (returning only strip rows) while the
    GPU estimates decoded chunks; wall clock including the decode (the step a
    user runs).  PNG decode bound: the GPU estimate is ~1 ms of it."""
    import tempfile
    import torch
    from paper_2210_14771_b200 import labels
    d = tempfile.mkdtemp(prefix="eca_labels_")
    for k in range(LABEL_FRAMES):
        labels.save_image(base[k % len(base)], os.path.join(d, f"frame_{k:05d}.png"))
    labels.pseudo_label(d, chunk=64)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    anns = labels.pseudo_label(d, chunk=64)
    dt = time.perf_counter() - t0
    return {"metric": "pseudo-labelled frames/s (§8f-1: PNG decode in worker processes + batched GPU estimate, "
                      "1080p; decode-bound)",
            "value": round(len(anns) / dt, 1), "unit": "frames/s", "frames": len(anns),
            "circles": int(sum(a.area is not None for a in anns)),
            "workers": max(1, min(32, os.cpu_count() or 1)),
            "note": "PNG decode bound (PIL, ~45 ms per 1080p frame per core): the GPU estimate is <1 % of "
                    "the wall clock; the CPU port decodes on every core and estimates inline", "_dir": d}


_CPU_LABEL_DIR = None


def _cpu_label(k: int):
    from PIL import Image
    from oracle import eca_oracle as orc
    from paper_2210_14771_b200.params import EcaConfig
    files = sorted(os.listdir(_CPU_LABEL_DIR))
    with Image.open(os.path.join(_CPU_LABEL_DIR, files[k % len(files)])) as im:
        frame = np.asarray(im.convert("RGB"))
    return orc.estimate(frame, EcaConfig(), 0)[0]


def label_cpu(d) -> dict:
    """The reference's pseudo_label per frame (PIL decode + estimate) through
    the oracle port, a process pool over the host cores, a bounded sample."""
    global _CPU_LABEL_DIR
    _CPU_LABEL_DIR = d
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    import multiprocessing as mp
    with ProcessPoolExecutor(cores, mp_context=mp.get_context("fork")) as ex:
        list(ex.map(_cpu_label, range(cores)))
        n = cores * 8
        t0 = time.perf_counter()
        list(ex.map(_cpu_label, range(n)))
        dt = time.perf_counter() - t0
    return {"value": round(n / dt, 2), "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": f"{n} PNG frames (1080p C2 mix): PIL decode + oracle-port estimate, process pool of {cores}"}


TRAIN_M, TRAIN_BATCH = 2048, 8


def _train_data(m: int):
    rng = np.random.default_rng(77)
    x = rng.normal(0.0, 1.0, (m, 5, 7, WIDTH)).astype(np.float32)
    t = rng.uniform(0.0, 1.0, (m, 1, 1, WIDTH - 6)).astype(np.float32)
    return x, t


def train_graph_step_us(eb, dev, xd, td, reps: int = 10) -> float:
    """Device time of one SGD step (forward + loss + backward + update, batch
    8): an epoch of 256 steps captured as one CUDA graph through the trainer's
    own calls, replayed `reps` times between CUDA events."""
    import ctypes
    import torch
    from paper_2210_14771_b200 import training as tr
    n, b = TRAIN_M, TRAIN_BATCH
    trn = tr._Trainer(eb.EdgeNet(eb.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=0), 7, WIDTH, b, dev)
    order = torch.from_numpy(np.random.default_rng(0).permutation(n).astype(np.int32)).to(dev)
    losses = torch.zeros(n // b, dtype=torch.float64, device=dev)

    def epoch():
        for k in range(n // b):
            idx = ctypes.c_void_p(order.data_ptr() + 4 * k * b)
            trn.forward(xd, idx, b)
            trn.backward(xd, td, idx, b, losses[k:k + 1])
            trn.sgd(1e-4)

    epoch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        epoch()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / (reps * (n // b))


def train_leg(eb, dev) -> dict:
    """§8f-4: EdgeNet SGD training (edgenet.train) over 2048 synthetic RGBXY
    strips (5 x 7 x 1920, the learned variant's input) in batches of 8,
    forward + BCE + backward + update on the GPU.  value: wall clock of the
    public call over 16 epochs with the strips resident in HBM (its first
    epoch runs eagerly, the second is captured as a CUDA graph, the rest
    replay it); device_us_per_step: one step of a replayed epoch graph, CUDA
    events."""
    import torch
    from paper_2210_14771_b200 import training as tr
    x, t = _train_data(TRAIN_M)
    xd, td = torch.from_numpy(x).to(dev), torch.from_numpy(t).to(dev)
    net = eb.EdgeNet(eb.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=0)
    tr.train(net, (xd[:64], td[:64]), None, tr.TrainConfig(learning_rate=0.001, batch_size=TRAIN_BATCH,
                                                            max_epochs=4))   # warm-up
    epochs = 16
    cfg = tr.TrainConfig(learning_rate=0.001, batch_size=TRAIN_BATCH, max_epochs=epochs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr.train(eb.EdgeNet(eb.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=0), (xd, td), None, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev_us = train_graph_step_us(eb, dev, xd, td)
    per_epoch = TRAIN_M // TRAIN_BATCH
    simt = os.environ.get("ECA_TRAIN_SIMT") == "1"
    return {"metric": "EdgeNet training samples/s (§8f-4: SGD epochs, batch 8 strips of 5x7x1920, "
                      "forward + BCE + backward + update)",
            "value": round(epochs * TRAIN_M / wall, 1), "unit": "samples/s",
            "ms_per_step": round(1e3 * wall / (epochs * per_epoch), 4),
            "device_us_per_step": round(dev_us, 1),
            "device_samples_per_s": round(TRAIN_BATCH / dev_us * 1e6, 1),
            "steps": epochs * per_epoch, "epochs": epochs,
            "launches_per_step": 16 if simt else 10,
            "kernels": "SIMT FP32 (ECA_TRAIN_SIMT=1)" if simt else
                       "tcgen05 3xTF32 conv forward / dgrad / wgrad (eca_train_tc.cuh)",
            "dtype": "f32", "data": "synthetic normal strips",
            "method": "value: wall clock of edgenet.train over 16 epochs of 2048 strips resident in HBM "
                      "(epoch 1 eager, epoch 2 captured as a CUDA graph, then replays); device: CUDA events "
                      "around 10 replays of a captured 256-step epoch"}


_CPU_TRAIN = None


def _cpu_train(k: int):
    from oracle import eca_oracle as orc
    x, t, layers = _CPU_TRAIN
    s = (k * TRAIN_BATCH) % (len(x) - TRAIN_BATCH)
    return orc.train_step(x[s:s + TRAIN_BATCH], t[s:s + TRAIN_BATCH], layers, 0.001)[0]


def train_cpu() -> dict:
    """The reference's training step (numpy im2col forward/backward, edgenet.py
    :100-130, 306-328) restated in the oracle, a process pool over the host
    cores, a bounded sample of steps."""
    global _CPU_TRAIN
    from oracle import eca_oracle as orc
    x, t = _train_data(64)
    _CPU_TRAIN = (x, t, orc.glorot_layers(0))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    import multiprocessing as mp
    with ProcessPoolExecutor(cores, mp_context=mp.get_context("fork")) as ex:
        list(ex.map(_cpu_train, range(cores)))
        n = cores * 2
        t0 = time.perf_counter()
        list(ex.map(_cpu_train, range(n)))
        dt = time.perf_counter() - t0
    return {"value": round(n * TRAIN_BATCH / dt, 2), "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": f"{n} SGD steps of 8 strips (5x7x1920) through the numpy oracle port of "
                      f"edgenet.train, process pool of {cores}, 1 BLAS thread each (independent steps)"}


def _records_np(rec):
    r = rec.cpu().numpy()
    i32 = r.view(np.int32).reshape(len(r), 10)
    return [(row[0], row[1], row[2], row[3], int(i[8]), int(i[9])) for row, i in zip(r, i32)]


_CPU_PAIRS = None


def _cpu_eval(idx: int):
    from oracle import eca_oracle as orc
    p, t = _CPU_PAIRS[idx % len(_CPU_PAIRS)]
    return orc.area_error_px_kdtree(p, t, WIDTH, HEIGHT)


def eval_cpu(pairs) -> dict:
    """The reference's evaluation algorithm on the host cores (boundary_points +
    cKDTree Hausdorff, metrics.py:148-223), a process pool, a bounded sample."""
    global _CPU_PAIRS
    _CPU_PAIRS = pairs
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    import multiprocessing as mp
    with ProcessPoolExecutor(cores, mp_context=mp.get_context("fork")) as ex:
        list(ex.map(_cpu_eval, range(cores)))
        n = max(len(pairs), cores * 16)
        t0 = time.perf_counter()
        list(ex.map(_cpu_eval, range(n), chunksize=4))
        dt = time.perf_counter() - t0
    return {"value": round(n / dt, 2), "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": f"{n} (fitted record, truth) pairs of the C2 1080p mix, oracle boundary_points + "
                      f"scipy cKDTree as metrics.py, process pool of {cores}"}


def uhd_leg(eb, dev, peaks) -> dict:
    """BASELINE config 4: 3840x2160 frames (the C2 mix rendered at 4K), 128 per
    step (4096 half-row items: the GPU's 2368 bound-and-prune warps stay busy),
    through the same streamed path, frames resident in HBM (12.7 GB pool)."""
    import torch
    from support import synth
    from paper_2210_14771_b200.engine import ContentAreaEngine
    w, h, b = 3840, 2160, 128
    specs = synth.bench_specs(8, w, h, seed=2024)
    base = torch.from_numpy(np.stack([synth.render(sp, 40000 + k) for k, (_, sp) in enumerate(specs)])).to(dev)
    slots = 4
    pool = torch.empty((slots * b, h, w, 3), dtype=torch.uint8, device=dev)   # 6.4 GB
    for i in range(slots * b):
        pool[i].copy_(base[i % len(base)])
    del base
    eng = ContentAreaEngine(h, w, b, device=dev)
    stream = torch.cuda.current_stream(dev)
    eng.run_stream(pool, 0, 3)
    eng.fence()
    steps = 40
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    eng.run_stream(pool, 3, steps)
    eng.fence(stream)
    e.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(e) / steps
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(4):
        eng.bounds(pool[(i % slots) * b:(i % slots + 1) * b], overlap=True, slot=i % 4)
    torch.cuda.synchronize()
    k0.record(stream)
    for i in range(steps):   # the pipeline's launch mode, as the 1080p roofline
        eng.bounds(pool[(i % slots) * b:(i % slots + 1) * b], overlap=True, slot=i % 4)
    k1.record(stream)
    torch.cuda.synchronize()
    k_ms = k0.elapsed_time(k1) / steps
    nbytes = b * eng.n_strips * 3 * w * 3
    gbs = nbytes / (k_ms * 1e-3) / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    del pool
    torch.cuda.empty_cache()
    return {"metric": "4K frames/s (3840x2160, C2 mix rendered at 4K, 128 per step, streamed)",
            "value": round(b / (ms * 1e-3), 1), "unit": "frames/s", "ms_per_step": round(ms, 5),
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "kernel": "eca::bounds_kernel<1, 0>",
                         "kernel_ms": round(k_ms, 5), "algorithmic_bytes_per_launch": nbytes,
                         "launch_mode": "back to back with programmatic dependent launch, 4 workspaces"}}


def latency(eb, dev) -> dict:
    """Single-frame (C1 1080p) latency.  Device: CUDA-graph replay of the one
    fused launch, CUDA events per replay.  Host: wall clock of the public
    estimate() on a CUDA tensor and on a numpy frame (result on the host)."""
    import torch
    from support import synth
    from paper_2210_14771_b200.engine import ContentAreaEngine
    frame = synth.c1_frame()
    t = torch.from_numpy(frame).to(dev).unsqueeze(0)
    eng = ContentAreaEngine(HEIGHT, WIDTH, 1, device=dev)
    eng.capture(t)
    stream = torch.cuda.current_stream(dev)
    for _ in range(50):
        eng.replay()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(1000)]
    for a, b in evs:
        a.record(stream)
        eng.replay()
        b.record(stream)
    torch.cuda.synchronize()
    times = sorted(a.elapsed_time(b) for a, b in evs)
    pct = lambda v, q: v[min(len(v) - 1, int(math.ceil(q * len(v))) - 1)]  # noqa: E731
    out = {"p50": round(pct(times, 0.50), 5), "p99": round(pct(times, 0.99), 5),
           "mean": round(sum(times) / len(times), 5), "runs": len(times),
           "method": "C1 1080p frame, CUDA graph replay of the fused launch, CUDA events per replay"}
    t3 = t[0]
    for name, src in (("cuda", t3), ("numpy", frame)):
        for _ in range(50):
            eb.estimate(src)
        host = []
        for _ in range(1000):
            w = time.perf_counter()
            eb.estimate(src)
            host.append((time.perf_counter() - w) * 1e3)
        host.sort()
        out[f"api_{name}_p50"] = round(pct(host, 0.5), 4)
        out[f"api_{name}_p99"] = round(pct(host, 0.99), 4)
    out["api_method"] = ("wall clock of eb.estimate(frame) -> ContentArea on the host, 1000 calls: a (H,W,3) "
                         "CUDA tensor, and a numpy frame (strip rows staged in pinned memory, read by the kernel "
                         "over PCIe)")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
