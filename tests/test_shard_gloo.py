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
