"""The NCCL record gather and the frame-sharded estimator on the GPU box's
single GPU (world size 1 over NCCL: the same code path the 2/4/8-GPU bench
takes, minus the peers; the N > 1 exchange is covered by the gloo world-2
tests)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2210_14771_b200 as eb
from support import synth
from paper_2210_14771_b200.shard import ShardedEstimator, gather_records

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def nccl_world1():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_sharded_estimator_nccl_matches_run(nccl_world1):
    specs = synth.bench_specs(10, 640, 480, seed=3)
    frames = torch.from_numpy(np.stack([synth.render(s, 500 + k) for k, (_, s) in enumerate(specs)])).cuda()
    se = ShardedEstimator(10, 480, 640, chunk=4)   # two full chunks and a ragged tail
    got = se.run(frames)
    want = torch.cat([eb.ContentAreaEngine(480, 640, 10).run(frames)])
    torch.cuda.synchronize()
    assert got.shape == (10, 5)
    assert torch.equal(got, want)


def test_gather_records_nccl(nccl_world1):
    rec = torch.arange(35, dtype=torch.float64, device="cuda").view(7, 5)
    out = gather_records(rec, 7)
    assert torch.equal(out, rec)


def test_sharded_estimator_pipelined_chunks(nccl_world1):
    """Batches of 32 through the pipeline (two launches per batch, records
    written by the fit kernel into the send buffer, gathers every 2 batches
    on the side stream) plus a fused ragged tail, vs one batched estimate."""
    specs = synth.bench_specs(20, 640, 480, seed=8)
    base = torch.from_numpy(np.stack([synth.render(s, 600 + k) for k, (_, s) in enumerate(specs)])).cuda()
    frames = base[[k % 20 for k in range(100)]].contiguous()
    se = ShardedEstimator(100, 480, 640, chunk=32, gather_every=2)
    assert not se.engine.fused and se.tail_engine.fused
    got = se.run(lambda a, b: frames[a:b], frames_ready=True)
    want = eb.ContentAreaEngine(480, 640, 100).run(frames)
    torch.cuda.synchronize()
    assert se.gathers == 2
    assert torch.equal(got, want)
