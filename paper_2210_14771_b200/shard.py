"""Frame-sharded multi-GPU estimation: one process per GPU, no data-path exchange.

Frames are independent (estimate() is a pure per-frame function and
estimate_batch reuses one seed for every frame, estimator.py:85-111), so a
stream of frames shards by contiguous frame ranges (BASELINE
config 5).  Each rank streams its range through the pipelined engine (one
bound-and-prune launch + one fit launch per batch, ContentAreaEngine.
run_pipelined) and the only collective is an all-gather of the 40-byte
EcaFitRecord per frame, issued per chunk of batches on a separate stream so it
overlaps the next batches (NCCL over NVLink on B200 boxes, gloo in CPU tests).
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

RECORD_DOUBLES = 5   # EcaFitRecord = 4 doubles + 2 int32


def shard_range(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) of frames owned by ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_capacity(n_frames: int, world: int) -> int:
    """Rows every rank sends per gather (the largest shard; smaller ones pad)."""
    return -(-n_frames // world)


def assemble(parts: torch.Tensor, n_frames: int, world: int) -> torch.Tensor:
    """(world, cap, 5) per-rank record blocks -> the (n_frames, 5) table in frame order."""
    rows = []
    for r in range(world):
        a, b = shard_range(n_frames, r, world)
        rows.append(parts[r, :b - a])
    return torch.cat(rows)


def gather_records(local: torch.Tensor, n_frames: int, group=None) -> torch.Tensor:
    """All-gather per-rank (n_local, 5) float64 record blocks into the full
    (n_frames, 5) table in frame order (every rank receives it)."""
    world = _rank_world(group)[1]
    if local.dim() != 2 or local.shape[1] != RECORD_DOUBLES or local.dtype != torch.float64:
        raise ValueError("records must be (n, 5) float64 EcaFitRecord rows")
    cap = shard_capacity(n_frames, world)
    send = torch.zeros((cap, RECORD_DOUBLES), dtype=torch.float64, device=local.device)
    send[:local.shape[0]] = local
    return assemble(_all_gather(send, world, group), n_frames, world)


def _rank_world(group=None) -> tuple[int, int]:
    """(rank, world) of the group; a single process without a process group is (0, 1)."""
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _all_gather(send: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """(rows, 5) from every rank -> (world, rows, 5)."""
    if world == 1 and not dist.is_initialized():
        return send.unsqueeze(0).clone()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * send.shape[0], RECORD_DOUBLES), dtype=send.dtype, device=send.device)
        dist.all_gather_into_tensor(out, send, group=group)
        return out.view(world, send.shape[0], RECORD_DOUBLES)
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    return torch.stack(parts)


class ShardedEstimator:
    """estimate() over a stream of ``n_frames`` frames split across the ranks
    of the default group (BASELINE config 5).

    Each rank owns the contiguous range ``shard_range(n_frames, rank, world)``
    and streams it in batches of ``chunk`` frames through ONE pipelined engine
    (plus one engine for a ragged tail, both built once); the fit of every
    batch writes its records straight into this rank's slice of a send buffer.
    Every ``gather_every`` batches the finished slice is all-gathered on a
    separate stream (it overlaps the next batches).  ``run`` returns the
    (n_frames, 5) records table in frame order on every rank.

    ``engine_factory(batch)`` builds an engine with ``run_pipelined(frames,
    frames_ready=..., records_out=...)`` and ``fence()`` (the default is a
    ContentAreaEngine; tests pass a stub).
    """

    def __init__(self, n_frames: int, height: int, width: int, cfg=None, seed: int = 0,
                 device=None, chunk: int = 256, gather_every: int = 32,
                 engine_factory: Callable | None = None, group=None):
        self.group = group
        self.rank, self.world = _rank_world(group)
        self.n_frames = n_frames
        self.start, self.stop = shard_range(n_frames, self.rank, self.world)
        self.n_local = self.stop - self.start
        self.cap = shard_capacity(n_frames, self.world)
        self.chunk = chunk
        self.gather_every = max(1, gather_every)
        if engine_factory is None:
            from .engine import ContentAreaEngine

            def engine_factory(b):
                return ContentAreaEngine(height, width, b, cfg=cfg, seed=seed, device=device)
        self.engine = engine_factory(chunk) if self.n_local >= chunk else None
        tail = self.n_local % chunk
        self.tail_engine = engine_factory(tail) if tail else None
        ref = self.engine or self.tail_engine
        if ref is not None and hasattr(ref, "device"):
            self.device = torch.device(ref.device)
        elif device is not None:
            self.device = torch.device(device)
        else:   # an empty shard still joins the collectives
            self.device = torch.device("cuda", torch.cuda.current_device()) \
                if dist.is_initialized() and dist.get_backend(group) == "nccl" else torch.device("cpu")
        self.send = torch.zeros((self.cap, RECORD_DOUBLES), dtype=torch.float64, device=self.device)
        self.cuda = self.device.type == "cuda"
        self.gather_stream = torch.cuda.Stream(self.device) if self.cuda else None
        self.gathers = 0

    def batches(self) -> list[tuple[int, int]]:
        """[a, b) local row ranges of the batches, in order."""
        return [(a, min(self.n_local, a + self.chunk)) for a in range(0, self.n_local, self.chunk)]

    def _gather_rows(self, a: int, b: int, outs: list) -> None:
        """All-gather rows [a, b) of every rank's send buffer (after this rank's
        stream has produced them)."""
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            self.gather_stream.wait_event(ev)
            with torch.cuda.stream(self.gather_stream):
                outs.append((a, b, _all_gather(self.send[a:b], self.world, self.group)))
        else:
            outs.append((a, b, _all_gather(self.send[a:b], self.world, self.group)))
        self.gathers += 1

    def gather_spans(self) -> list[tuple[int, int]]:
        """Row ranges of the gathers: the same on every rank (they are
        collectives), cut from the largest shard; smaller shards send padding."""
        step = self.gather_every * self.chunk
        return [(g, min(self.cap, g + step)) for g in range(0, self.cap, step)] or [(0, 0)]

    def run(self, frames: Callable[[int, int], torch.Tensor] | torch.Tensor,
            frames_ready: bool = False) -> torch.Tensor:
        """frames: this rank's shard as a (n_local, H, W, 3) tensor, or a callable
        (a, b) -> the frames of local rows [a, b) (e.g. views into a pool).
        frames_ready: the frames were complete before this call (see
        ContentAreaEngine.run_pipelined)."""
        get = frames if callable(frames) else (lambda a, b: frames[a:b])
        outs: list = []
        spans = self.gather_spans()
        gi = 0

        def flush(upto: int) -> None:
            nonlocal gi
            if gi < len(spans) and spans[gi][1] <= upto:
                for e in (self.engine, self.tail_engine):
                    if e is not None:
                        e.fence()
            while gi < len(spans) and spans[gi][1] <= upto:
                self._gather_rows(*spans[gi], outs)
                gi += 1

        for a, b in self.batches():
            eng = self.engine if b - a == self.chunk else self.tail_engine
            eng.run_pipelined(get(a, b), frames_ready=frames_ready, records_out=self.send[a:b])
            flush(b)
        flush(self.cap)   # the rest (this shard may be one row short of the largest)
        if self.cuda:
            torch.cuda.current_stream(self.device).wait_stream(self.gather_stream)
        parts = torch.empty((self.world, self.cap, RECORD_DOUBLES), dtype=torch.float64, device=self.device)
        for a, b, p in outs:
            parts[:, a:b] = p
        return assemble(parts, self.n_frames, self.world)
