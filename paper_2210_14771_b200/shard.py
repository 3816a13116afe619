"""Frame-sharded multi-GPU estimation: one process per GPU, no data-path exchange.

Frames are independent (estimate() is a pure per-frame function and
estimate_batch reuses one seed for every frame, estimator.py:85-111), so a
batch or stream shards by contiguous frame ranges; each rank runs the fused
kernel on its shard and the only collective is an all-gather of the 40-byte
EcaFitRecord per frame (NCCL over NVLink on B200 boxes, gloo in CPU tests).
"""

from __future__ import annotations

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


def gather_records(local: torch.Tensor, n_frames: int, group=None) -> torch.Tensor:
    """All-gather per-rank (n_local, 5) float64 record blocks into the full
    (n_frames, 5) table in frame order (every rank receives it)."""
    world = dist.get_world_size(group)
    if local.dim() != 2 or local.shape[1] != RECORD_DOUBLES or local.dtype != torch.float64:
        raise ValueError("records must be (n, 5) float64 EcaFitRecord rows")
    cap = -(-n_frames // world)            # ceil: every rank sends the same size
    send = torch.zeros((cap, RECORD_DOUBLES), dtype=torch.float64, device=local.device)
    send[:local.shape[0]] = local
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * cap, RECORD_DOUBLES), dtype=torch.float64, device=local.device)
        dist.all_gather_into_tensor(out, send, group=group)
        parts = list(out.view(world, cap, RECORD_DOUBLES))
    else:
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send, group=group)
    rows = []
    for r in range(world):
        a, b = shard_range(n_frames, r, world)
        rows.append(parts[r][:b - a])
    return torch.cat(rows)


class ShardedEstimator:
    """estimate() over a frame set split across the ranks of the default group.

    ``run(frames_local)`` takes this rank's shard on its GPU and returns the
    gathered (n_frames, 5) records on every rank.
    """

    def __init__(self, n_frames: int, height: int, width: int, cfg=None, seed: int = 0,
                 device=None, chunk: int = 256):
        from .engine import ContentAreaEngine
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.n_frames = n_frames
        self.start, self.stop = shard_range(n_frames, self.rank, self.world)
        self.chunk = chunk
        self.engine = ContentAreaEngine(height, width, chunk, cfg=cfg, seed=seed, device=device)
        self.device = self.engine.device

    def run(self, frames_local: torch.Tensor) -> torch.Tensor:
        n = self.stop - self.start
        if frames_local.shape[0] != n:
            raise ValueError(f"rank {self.rank} owns {n} frames, got {frames_local.shape[0]}")
        out = torch.empty((n, RECORD_DOUBLES), dtype=torch.float64, device=self.device)
        for a in range(0, n, self.chunk):
            b = min(n, a + self.chunk)
            if b - a == self.chunk:
                out[a:b] = self.engine.run(frames_local[a:b])
            else:   # ragged tail: a one-off engine of the tail size
                from .engine import ContentAreaEngine
                tail = ContentAreaEngine(self.engine.height, self.engine.width, b - a,
                                         cfg=self.engine.cfg, seed=self.engine.seed,
                                         device=self.device)
                out[a:b] = tail.run(frames_local[a:b])
        return gather_records(out, self.n_frames)
