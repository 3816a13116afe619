"""Programmatic dependent launch of back-to-back bound-and-prune kernels on K
rotating workspaces: time per launch and whether every launch's candidates
equal a serial reference run (so the overlap is measured only where it is
correct).  Also: the same with an event record after every launch (as
eca_pipeline_step has), to see whether the record breaks the overlap."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2210_14771_b200 as eb  # noqa: E402
from paper_2210_14771_b200 import _lib, api  # noqa: E402

B = 256
dev = torch.device('cuda', 0)
base = torch.from_numpy(bench.base_frames(40)).to(dev)
NP = 2048
pool = torch.empty((NP, 1080, 1920, 3), dtype=torch.uint8, device=dev)
for i in range(NP):
    pool[i].copy_(base[i % 40])
eng = eb.ContentAreaEngine(1080, 1920, B, device=dev)
lib = _lib.load()
st = api._stream(dev)
S = eng.n_strips
nslot = NP // B
K = 4
ws = [torch.zeros_like(eng.workspace) for _ in range(K)]
outs = [torch.zeros((B, 2 * S), dtype=torch.int32, device=dev) for _ in range(K)]
outy = [torch.zeros((B, 2 * S), dtype=torch.int32, device=dev) for _ in range(K)]
outs_s = [torch.zeros((B, 2 * S), dtype=torch.float64, device=dev) for _ in range(K)]


def bounds(i, flags, k):
    f = pool[(i % nslot) * B:][:B]
    _lib.check(lib.eca_bounds_handcrafted(api._ptr(f), B, f.stride(0), f.stride(1), eng._rows, None, S,
                                          ctypes.byref(eng.params), api._ptr(outs[k]), api._ptr(outy[k]),
                                          api._ptr(outs_s[k]), api._ptr(ws[k]), flags, st), "b")


def rescore(k):
    _lib.check(lib.eca_rescore_handcrafted(B, eng._rows, S, ctypes.byref(eng.params), api._ptr(outs[k]),
                                           api._ptr(outy[k]), api._ptr(outs_s[k]), api._ptr(ws[k]), st), "r")


# reference candidates per pool slot (serial launches + rescore)
ref = []
for j in range(nslot):
    bounds(j, 0, 0)
    rescore(0)
    torch.cuda.synchronize()
    ref.append((outs[0].clone(), outs_s[0].clone()))


def run(flags, nws, n=200, event=False):
    evs = [torch.cuda.Event() for _ in range(n)] if event else None
    for i in range(8):
        bounds(i, flags, i % nws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        bounds(i, flags, i % nws)
        if event:
            evs[i].record()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    # correctness of the last nws launches: survivor slots + counts equal the serial run
    ok = True
    for i in range(n - nws, n):
        k = i % nws
        rescore(k)
        torch.cuda.synchronize()
        ok &= bool(torch.equal(outs[k], ref[i % nslot][0])) and bool(torch.equal(outs_s[k], ref[i % nslot][1]))
    return us, ok


for flags, nws, ev in ((0, 1, False), (1, 2, False), (1, 3, False), (1, 4, False), (1, 3, True),
                       (3, 3, False), (0, 1, False)):
    us, ok = run(flags, nws, event=ev)
    print(f"flags={flags} workspaces={nws} event={ev}: {us:6.1f} us/launch  "
          f"{B * 16 * 3 * 1920 * 3 / us / 1e3:7.1f} GB/s  correct={ok}")
