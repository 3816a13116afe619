import sys, ctypes, numpy as np, torch, os
sys.path.insert(0, '.')
print("start", flush=True)
import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import _lib, api, synth
lib = _lib.load(); print("loaded", flush=True)
frame = synth.render(synth.bench_spec("clean", np.random.default_rng(1), 320, 240), 3)
t = torch.from_numpy(frame).cuda().unsqueeze(0); torch.cuda.synchronize(); print("frame on gpu", flush=True)
rows = eb.strip_heights(240, 16, 8.0); print(rows, flush=True)
xs = torch.empty((1, 32), dtype=torch.int32, device='cuda'); ys = torch.empty_like(xs); sc = torch.empty((1,32), dtype=torch.float64, device='cuda')
print("alloc", flush=True)
p = eb.EcaConfig().device_params(320, 240); print("params", flush=True)
b = ctypes.c_double(); print("bound", lib.eca_prefilter_bound(ctypes.byref(p), ctypes.byref(b)), b.value, flush=True)
ra = api._i32_array(rows); st = api._stream(t.device); print("args", st, flush=True)
os.environ["ECA_TRACE"] = "1"
rc = lib.eca_points_handcrafted(api._ptr(t), 1, t.stride(0), t.stride(1), ra, None, 16, ctypes.byref(p), api._ptr(xs), api._ptr(ys), api._ptr(sc), st)
print("rc", rc, flush=True)
torch.cuda.synchronize(); print("synced", flush=True)
print(xs.cpu().numpy(), flush=True)
