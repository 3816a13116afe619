"""N>1 path on CPU: frame sharding and the record all-gather with gloo, world size 2
(the GPU runs use NCCL; the exchange logic is identical)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_14771_b200.shard import gather_records, shard_range


def test_shard_range_covers_every_frame_once():
    for n in [0, 1, 7, 256, 100_000]:
        for world in [1, 2, 3, 4, 8]:
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_frames, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard_range(n_frames, rank, world)
        # synthetic per-frame records: cx = frame index, status in the int slot
        rec = torch.zeros((b - a, 5), dtype=torch.float64)
        rec[:, 0] = torch.arange(a, b, dtype=torch.float64)
        rec[:, 3] = 0.5 * torch.arange(a, b, dtype=torch.float64)
        rec.view(torch.int32).view(b - a, 10)[:, 9] = torch.arange(a, b, dtype=torch.int32) % 4
        full = gather_records(rec, n_frames)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [5, 8, 1])
def test_gather_records_world2(n_frames):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        full = out[r]
        assert full.shape == (n_frames, 5)
        assert np.array_equal(full[:, 0], np.arange(n_frames))
        assert np.array_equal(full[:, 3], 0.5 * np.arange(n_frames))
        assert np.array_equal(full.view(np.int32).reshape(n_frames, 10)[:, 9], np.arange(n_frames) % 4)
    assert np.array_equal(out[0], out[1])


class _StubEngine:
    """Stands in for ContentAreaEngine on CPU: 'frames' are global frame
    indices; the records it writes encode them."""

    def __init__(self, batch, log):
        self.batch, self.log = batch, log
        self.device = torch.device("cpu")

    def run_pipelined(self, frames, frames_ready=False, records_out=None):
        assert frames.shape[0] == self.batch and records_out.shape == (self.batch, 5)
        records_out.zero_()
        records_out[:, 0] = frames.double()
        records_out[:, 3] = 0.25 * frames.double()
        records_out.view(torch.int32).view(self.batch, 10)[:, 9] = (frames % 4).int()
        self.log.append(("run", self.batch))
        return records_out

    def fence(self):
        self.log.append(("fence", self.batch))


def _sharded_worker(rank, world, port, n_frames, chunk, every, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_14771_b200.shard import ShardedEstimator
        log = []
        est = ShardedEstimator(n_frames, 8, 8, chunk=chunk, gather_every=every,
                               engine_factory=lambda b: _StubEngine(b, log))
        idx = torch.arange(est.start, est.stop)
        full = est.run(lambda a, b: idx[a:b], frames_ready=True)
        n_eng = (est.engine is not None) + (est.tail_engine is not None)
        q.put((rank, full.numpy(), est.gathers, len(est.gather_spans()), n_eng,
               sum(1 for k, _ in log if k == "run"), len(est.batches())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("n_frames,chunk,every", [(100, 8, 2), (37, 8, 1), (3, 4, 2)])
def test_sharded_estimator_stream(world, n_frames, chunk, every):
    """ShardedEstimator over world 2 and 4 (gloo): contiguous shards, one
    engine per batch size (full + ragged tail) built once, the same gather
    schedule on every rank (collectives), the full table in frame order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, n_frames, chunk, every, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {r: rest for r, *rest in (q.get(timeout=180) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        full, gathers, spans, n_eng, runs, batches = out[r]
        assert full.shape == (n_frames, 5)
        assert np.array_equal(full[:, 0], np.arange(n_frames))
        assert np.array_equal(full[:, 3], 0.25 * np.arange(n_frames))
        assert np.array_equal(full.view(np.int32).reshape(n_frames, 10)[:, 9], np.arange(n_frames) % 4)
        assert gathers == spans == out[0][2]
        assert runs == batches and n_eng <= 2
