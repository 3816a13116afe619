"""Fixed-shape batched estimator: preallocated buffers, CUDA-graph replay and
strip-rows-only host ingest.  This is the throughput / latency path the bench
drives; the list-based API in ``api.py`` is built from the same calls.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, api
from .params import EcaConfig, config_default


class ContentAreaEngine:
    """estimate() for batches of ``batch`` frames of one (height, width).

    ``run(frames)``      frames already on the GPU (B,H,W,3) uint8 -> (B,5) records
    ``run_host(frames)`` pinned host frames: H2D of the strip rows only, one
                         fused launch, D2H of the 40-byte records
    ``capture(frames)``  record a CUDA graph of run(frames) for ``replay()``
    Records are EcaFitRecord rows (cx, cy, r, score, inliers|status).
    """

    def __init__(self, height: int, width: int, batch: int, cfg: EcaConfig | None = None,
                 seed: int = 0, variant: api.EstimatorVariant = api.HANDCRAFTED, device=None,
                 tensor_cores: bool = True):
        self.cfg = cfg or config_default()
        self.height, self.width, self.batch = height, width, batch
        self.device = api._device(device)
        self.variant = variant
        self.seed = seed
        # learned variant: the 3x3 layers on tcgen05 (default) or the SIMT kernel
        self.cnn_flags = 0 if tensor_cores else _lib.LEARNED_SIMT
        self.rows = api.strip_heights(height, self.cfg.strip_count, self.cfg.strip_weighting)
        s = self.n_strips = len(self.rows)
        self.half = api.HALF_WINDOW if isinstance(variant, api.Learned) else 1
        self._rows = api._i32_array(self.rows)
        self._first = api._i32_array([r - self.half for r in self.rows])
        rpb = 2 * self.half + 1
        self._band = api._i32_array([k * rpb for k in range(s)])
        self.params = self.cfg.device_params(width, height)
        d = self.device
        self.trip = api._dev_triplets(seed, self.cfg.ransac_attempts, 2 * s, d)
        self.counters = torch.zeros(max(batch, 64), dtype=torch.int32, device=d)
        self.xs = torch.empty((batch, 2 * s), dtype=torch.int32, device=d)
        self.ys = torch.empty_like(self.xs)
        self.sc = torch.empty((batch, 2 * s), dtype=torch.float64, device=d)
        self.rec = torch.empty((batch, 5), dtype=torch.float64, device=d)
        self.bands = torch.empty((batch, s * rpb, width, 3), dtype=torch.uint8, device=d)
        nws = ctypes.c_int64()
        _lib.check(_lib.load().eca_points_workspace_bytes(batch, s, ctypes.byref(nws)),
                   "eca_points_workspace_bytes")
        self.workspace = torch.zeros(max(nws.value, 256), dtype=torch.uint8, device=d)
        self._bounds_ws = [self.workspace]   # bounds(): extra slots made on demand
        self.rec_host = torch.empty((batch, 5), dtype=torch.float64, pin_memory=True)
        if isinstance(variant, api.Learned):
            self.probs = torch.empty((batch, s, width - 6), dtype=torch.float32, device=d)
            self.w_dev, self.norm = api._dev_net(variant.net, d)
        self.graph = None
        self._pipe = None
        self._pipe_graph = None
        # Small batches (latency): one fused launch whose last strip CTA per
        # frame runs the fit.  Large batches (throughput): one launch of the
        # bound-and-prune kernel (warp per half row) whose final stage -- the
        # warp that completes a frame's last half row -- rescores the frame's
        # survivors in FP64 and fits it.
        self.fused = batch <= self.FUSED_MAX_BATCH
        if isinstance(variant, api.Learned):
            self.launches_per_run = 3          # CNN, candidate select, fit
        else:
            self.launches_per_run = 1 if self.fused else 2   # fused | bounds, fit
        self.launches_per_step = self.launches_per_run   # run_pipelined: bounds + fit launches

    FUSED_MAX_BATCH = 16

    # ------------------------------------------------------------ launches
    def _launch(self, ptr: int, fstride: int, rstride: int, band) -> None:
        lib = _lib.load()
        st = api._stream(self.device)
        s = self.n_strips
        if isinstance(self.variant, api.Learned):
            rc = lib.eca_points_learned_ex(ctypes.c_void_p(ptr), self.batch, fstride, rstride, self._rows,
                                           band, s, self.height, self.width, api._ptr(self.w_dev),
                                           self.norm, self.cnn_flags, api._ptr(self.probs),
                                           api._ptr(self.xs), api._ptr(self.ys), api._ptr(self.sc), st)
            _lib.check(rc, "eca_points_learned_ex")
            rc = lib.eca_fit(api._ptr(self.xs), api._ptr(self.ys), api._ptr(self.sc), self.batch,
                             2 * s, ctypes.byref(self.params), api._ptr(self.trip), 0,
                             api._ptr(self.rec), st)
            _lib.check(rc, "eca_fit")
            return
        if self.fused:
            rc = lib.eca_estimate_handcrafted(ctypes.c_void_p(ptr), self.batch, fstride, rstride,
                                              self._rows, band, s, ctypes.byref(self.params),
                                              api._ptr(self.trip), api._ptr(self.counters),
                                              api._ptr(self.xs), api._ptr(self.ys),
                                              api._ptr(self.sc), api._ptr(self.rec), st)
            _lib.check(rc, "eca_estimate_handcrafted")
            return
        rc = lib.eca_estimate_batch_handcrafted(
            ctypes.c_void_p(ptr), self.batch, fstride, rstride, self._rows, band, s,
            ctypes.byref(self.params), api._ptr(self.trip), api._ptr(self.workspace), api._ptr(self.xs),
            api._ptr(self.ys), api._ptr(self.sc), api._ptr(self.rec), None, 0, st)
        _lib.check(rc, "eca_estimate_batch_handcrafted")

    def _check_frames(self, frames: torch.Tensor) -> torch.Tensor:
        if frames.dim() == 3:
            frames = frames.unsqueeze(0)
        if tuple(frames.shape) != (self.batch, self.height, self.width, 3) or frames.dtype != torch.uint8:
            raise ValueError(f"expected uint8 frames of shape {(self.batch, self.height, self.width, 3)}, "
                             f"got {tuple(frames.shape)} {frames.dtype}")
        if frames.stride(3) != 1 or frames.stride(2) != 3:
            frames = frames.contiguous()
        return frames

    def points(self, frames: torch.Tensor) -> None:
        """Only the strip-scoring kernel (candidates into self.xs/ys/sc); the
        bench times it alone for the roofline of the dominant kernel."""
        f = self._check_frames(frames)
        rc = _lib.load().eca_points_handcrafted(
            ctypes.c_void_p(f.data_ptr()), self.batch, f.stride(0), f.stride(1), self._rows, None,
            self.n_strips, ctypes.byref(self.params), api._ptr(self.xs), api._ptr(self.ys),
            api._ptr(self.sc), api._ptr(self.workspace), api._stream(self.device))
        _lib.check(rc, "eca_points_handcrafted")

    # ------------------------------------------------------------ pipeline
    def _pipeline(self):
        """The native streamed pipeline (eca_pipeline_*), created on first use."""
        if self._pipe is None:
            lib = _lib.load()
            n = ctypes.c_int64()
            _lib.check(lib.eca_pipeline_bytes(self.batch, self.n_strips, ctypes.byref(n)),
                       "eca_pipeline_bytes")
            scratch = torch.empty(n.value, dtype=torch.uint8, device=self.device)
            handle = ctypes.c_void_p()
            torch.cuda.synchronize(self.device)
            _lib.check(lib.eca_pipeline_create(self.batch, self.height, self.width, self._rows,
                                               self.n_strips, ctypes.byref(self.params),
                                               api._ptr(self.trip), api._ptr(scratch), n.value,
                                               ctypes.byref(handle)), "eca_pipeline_create")
            self._pipe = {"handle": handle, "scratch": scratch, "base": scratch.data_ptr(), "views": {},
                          "out": ctypes.c_void_p(), "step": lib.eca_pipeline_step}
        return self._pipe

    def _release_pipeline(self):
        self._pipe_graph = None
        if self._pipe is not None:
            _lib.load().eca_pipeline_destroy(self._pipe["handle"])
            self._pipe = None

    def __del__(self):
        try:
            self._release_pipeline()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    PIPE_SETS = 4   # eca_pipeline_* buffer sets (records stay valid this many steps)

    def run_pipelined(self, frames: torch.Tensor, frames_ready: bool = False,
                      records_out: torch.Tensor | None = None) -> torch.Tensor:
        """Throughput mode for a stream of batches: ONE launch per batch
        (eca_pipeline_step) on the current stream -- bound-and-prune with the
        final stage (each frame's last half-row warp rescores and fits it);
        consecutive launches overlap (programmatic dependent launch).  The
        returned (B,5) records are complete in current-stream order
        (``fence()`` for other streams) and are overwritten PIPE_SETS calls
        later.  ``frames_ready``: the frames were complete before the previous
        operation on the stream was enqueued (a pre-filled pool), so the
        kernel need not wait for that operation (otherwise it does, in case it
        produced them).  ``records_out``: a (B,5) float64 tensor (device or
        pinned host) the fit kernel also writes this batch's records to.  Same
        records as run() (tests/test_gpu_parity.py)."""
        if records_out is not None and (tuple(records_out.shape) != (self.batch, 5) or
                                        records_out.dtype != torch.float64 or
                                        not records_out.is_contiguous() or
                                        not (records_out.is_cuda or records_out.is_pinned())):
            raise ValueError("records_out must be a contiguous (B,5) float64 device or pinned tensor")
        if isinstance(self.variant, api.Learned) or self.fused:
            rec = self.run(frames)
            if records_out is not None:
                records_out.copy_(rec, non_blocking=True)
            return rec
        if frames.dim() == 4 and (frames.stride(3) != 1 or frames.stride(2) != 3):
            raise ValueError("run_pipelined takes frames with packed pixels (stride (.., .., 3, 1))")
        f = self._check_frames(frames)
        if f.device != self.device:
            raise ValueError(f"frames must live on {self.device}")
        p = self._pipeline()
        out = p["out"]
        flags = _lib.PIPE_FRAMES_READY if frames_ready else 0
        extra = None if records_out is None else ctypes.c_void_p(records_out.data_ptr())
        _lib.check(p["step"](p["handle"], ctypes.c_void_p(f.data_ptr()), f.stride(0), f.stride(1), flags,
                             extra, ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream),
                             ctypes.byref(out)), "eca_pipeline_step")
        return self._record_view(p, out.value)

    def run_stream(self, pool: torch.Tensor, first: int, steps: int, frames_ready: bool = True) -> list:
        """``steps`` run_pipelined calls in ONE native call (eca_pipeline_run):
        step j takes batch ((first + j) % n_batches) of ``pool``, a (n_batches *
        B, H, W, 3) device tensor.  Returns the record tensors of the last
        min(steps, PIPE_SETS) steps, oldest first (complete in current-stream
        order; valid until PIPE_SETS further steps)."""
        if isinstance(self.variant, api.Learned) or self.fused:
            raise ValueError("run_stream streams the handcrafted variant at batch > 16")
        if pool.dim() != 4 or pool.shape[0] % self.batch or tuple(pool.shape[1:]) != \
                (self.height, self.width, 3) or pool.dtype != torch.uint8 or not pool.is_contiguous():
            raise ValueError("pool must be a contiguous (n * B, H, W, 3) uint8 tensor")
        if pool.device != self.device:
            raise ValueError(f"pool must live on {self.device}")
        p = self._pipeline()
        lib = _lib.load()
        flags = _lib.PIPE_FRAMES_READY if frames_ready else 0
        _lib.check(lib.eca_pipeline_run(p["handle"], ctypes.c_void_p(pool.data_ptr()),
                                        self.batch * pool.stride(0), pool.shape[0] // self.batch, first,
                                        steps, pool.stride(0), pool.stride(1), flags,
                                        ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)),
                   "eca_pipeline_run")
        recs = []
        for back in range(min(steps, self.PIPE_SETS) - 1, -1, -1):
            _lib.check(lib.eca_pipeline_records(p["handle"], back, ctypes.byref(p["out"])), "eca_pipeline_records")
            recs.append(self._record_view(p, p["out"].value))
        return recs

    def _record_view(self, p, ptr: int) -> torch.Tensor:
        rec = p["views"].get(ptr)
        if rec is None:   # a view of this buffer set's records inside the scratch
            off = ptr - p["base"]
            rec = p["scratch"][off:off + self.batch * 40].view(torch.float64).view(self.batch, 5)
            p["views"][ptr] = rec
        return rec

    def run_host_pipelined(self, host_frames: torch.Tensor, host_records: torch.Tensor) -> None:
        """Streaming end-to-end mode: pinned host frames in, pinned host
        records out, no synchronisation.  One launch per call on the current
        stream: the bound-and-prune kernel reads the frames over PCIe chunk by
        chunk (zero-copy TMA), and the final stage stores each frame's record
        straight into ``host_records`` ((B,5) float64, pinned); calls overlap.
        Both buffers must stay untouched until the stream is synchronised."""
        a = host_frames
        if not isinstance(a, torch.Tensor) or a.is_cuda or not a.is_pinned():
            raise ValueError("run_host_pipelined takes a pinned host frame tensor")
        if tuple(a.shape) != (self.batch, self.height, self.width, 3) or a.dtype != torch.uint8 \
                or a.stride(3) != 1 or a.stride(2) != 3:
            raise ValueError("host frames must be (B,H,W,3) uint8 with packed pixels")
        r = host_records
        if r.is_cuda or not r.is_pinned() or tuple(r.shape) != (self.batch, 5) or r.dtype != torch.float64:
            raise ValueError("host_records must be a pinned (B,5) float64 tensor")
        if isinstance(self.variant, api.Learned) or self.fused:
            raise ValueError("run_host_pipelined streams the handcrafted variant at batch > 16")
        p = self._pipeline()
        # host frames were written before this call: nothing on the stream produces them
        _lib.check(p["step"](p["handle"], ctypes.c_void_p(a.data_ptr()), a.stride(0), a.stride(1),
                             _lib.BOUNDS_ZERO_COPY | _lib.PIPE_FRAMES_READY, ctypes.c_void_p(r.data_ptr()),
                             ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream),
                             ctypes.byref(p["out"])), "eca_pipeline_step")

    def capture_pipelined(self, batches, frames_ready: bool = True) -> None:
        """Record run_pipelined() over ``batches`` (device frame tensors whose
        storage stays put) plus the closing fence as ONE CUDA graph: both
        streams, the events between them and the programmatic-dependent
        bound-and-prune launches become graph nodes, so replay_pipelined()
        streams the whole sequence with one host call instead of one native
        call per batch (which bounds the step at ~28 us of host time).  The
        records of batch k are the ones run_pipelined returned for it during
        capture; the graph replays exactly that sequence."""
        p = self._pipe if self._pipe is not None else self._pipeline()
        torch.cuda.synchronize(self.device)
        _lib.check(_lib.load().eca_pipeline_reset(p["handle"]), "eca_pipeline_reset")
        g = torch.cuda.CUDAGraph()
        recs = []
        with torch.cuda.graph(g):
            for f in batches:
                recs.append(self.run_pipelined(f, frames_ready=frames_ready))
            self.fence()
        torch.cuda.synchronize(self.device)
        _lib.check(_lib.load().eca_pipeline_reset(p["handle"]), "eca_pipeline_reset")
        self._pipe_graph = (g, recs)

    def replay_pipelined(self) -> list:
        """Launch the captured pipeline graph on the current stream; returns
        the per-batch record tensors (complete when the stream reaches here)."""
        g, recs = self._pipe_graph
        g.replay()
        return recs

    def fence(self, stream: torch.cuda.Stream | None = None) -> None:
        """Make ``stream`` (default: current) wait for every run_pipelined() so far."""
        if self._pipe is None:
            return
        stream = stream or torch.cuda.current_stream(self.device)
        _lib.check(_lib.load().eca_pipeline_fence(self._pipe["handle"],
                                                  ctypes.c_void_p(stream.cuda_stream)),
                   "eca_pipeline_fence")

    def bounds(self, frames: torch.Tensor, overlap: bool = False, slot: int = 0) -> None:
        """Only the bound-and-prune kernel (the step's dominant kernel; its
        survivors land in workspace ``slot``): the bench's roofline timing.
        ``overlap``: programmatic dependent launch, as the streaming pipeline
        launches it; back-to-back overlapped launches need >= 3 rotating slots
        (a launch may still run while the next two start)."""
        f = self._check_frames(frames)
        while len(self._bounds_ws) <= slot:
            self._bounds_ws.append(torch.zeros_like(self.workspace))
        ws = self._bounds_ws[slot]
        _lib.check(_lib.load().eca_bounds_handcrafted(
            ctypes.c_void_p(f.data_ptr()), self.batch, f.stride(0), f.stride(1), self._rows, None,
            self.n_strips, ctypes.byref(self.params), api._ptr(self.xs), api._ptr(self.ys),
            api._ptr(self.sc), api._ptr(ws), _lib.BOUNDS_OVERLAP_PREVIOUS if overlap else 0,
            api._stream(self.device)), "eca_bounds_handcrafted")

    def run(self, frames: torch.Tensor) -> torch.Tensor:
        """Frames on this GPU -> device records (asynchronous)."""
        f = self._check_frames(frames)
        if f.device != self.device:
            raise ValueError(f"frames must live on {self.device}")
        self._launch(f.data_ptr(), f.stride(0), f.stride(1), None)
        return self.rec

    def ingest(self, host_frames) -> None:
        """Strip-row H2D copies of a pinned host batch into ``self.bands``."""
        a = host_frames
        if isinstance(a, torch.Tensor):
            if a.is_cuda:
                raise ValueError("ingest() takes host frames")
            ptr, fs, rs = a.data_ptr(), a.stride(0), a.stride(1)
            ok = a.stride(3) == 1 and a.stride(2) == 3
        else:
            ptr, fs, rs = a.ctypes.data, a.strides[0], a.strides[1]
            ok = a.strides[3] == 1 and a.strides[2] == 3
        if tuple(a.shape) != (self.batch, self.height, self.width, 3) or not ok:
            raise ValueError("host frames must be (B,H,W,3) uint8 with packed pixels")
        rc = _lib.load().eca_h2d_bands(ctypes.c_void_p(ptr), self.batch, fs, rs, self._first,
                                       self.n_strips, 2 * self.half + 1, self.width,
                                       api._ptr(self.bands), api._stream(self.device))
        _lib.check(rc, "eca_h2d_bands")

    def run_bands(self) -> torch.Tensor:
        self._launch(self.bands.data_ptr(), self.bands.stride(0), self.bands.stride(1), self._band)
        return self.rec

    def run_host(self, host_frames) -> torch.Tensor:
        """Pinned host frames -> pinned host records (synchronises the stream)."""
        self.ingest(host_frames)
        self.run_bands()
        self.rec_host.copy_(self.rec, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return self.rec_host

    def run_host_zero_copy(self, host_frames: torch.Tensor) -> torch.Tensor:
        """Pinned host frames -> pinned host records (synchronises the stream),
        without copying the frames: the bound-and-prune kernel reads the
        strip rows straight from pinned host memory over PCIe, scan chunk by
        scan chunk (ECA_BOUNDS_ZERO_COPY), so only the columns it visits cross
        the bus.  Handcrafted variant; same records as run()."""
        a = host_frames
        if not isinstance(a, torch.Tensor) or a.is_cuda or not a.is_pinned():
            raise ValueError("run_host_zero_copy takes a pinned host tensor")
        if tuple(a.shape) != (self.batch, self.height, self.width, 3) or a.dtype != torch.uint8 \
                or a.stride(3) != 1 or a.stride(2) != 3:
            raise ValueError("host frames must be (B,H,W,3) uint8 with packed pixels")
        if isinstance(self.variant, api.Learned):
            raise ValueError("zero-copy ingest is implemented for the handcrafted variant")
        lib = _lib.load()
        st = api._stream(self.device)
        _lib.check(lib.eca_estimate_batch_handcrafted(
            ctypes.c_void_p(a.data_ptr()), self.batch, a.stride(0), a.stride(1), self._rows, None,
            self.n_strips, ctypes.byref(self.params), api._ptr(self.trip), api._ptr(self.workspace),
            api._ptr(self.xs), api._ptr(self.ys), api._ptr(self.sc), api._ptr(self.rec),
            ctypes.c_void_p(self.rec_host.data_ptr()), _lib.BOUNDS_ZERO_COPY, st),
            "eca_estimate_batch_handcrafted")
        torch.cuda.current_stream(self.device).synchronize()
        return self.rec_host

    def pipeline_zero_copy_bytes(self) -> int:
        """Bytes the pipelined bound-and-prune launches fetched over PCIe in
        zero-copy mode so far (every buffer set's counter)."""
        if self._pipe is None:
            return 0
        sc = self._pipe["scratch"]
        per_set = sc.numel() // self.PIPE_SETS
        return int(sum(int(sc[k * per_set + 8:k * per_set + 12].view(torch.int32).item())
                       for k in range(self.PIPE_SETS))) * 16

    def zero_copy_bytes(self) -> int:
        """Bytes fetched over PCIe by run_host_zero_copy() calls so far."""
        return int(self.workspace[8:12].view(torch.int32).item()) * 16

    # --------------------------------------------------------------- graphs
    def capture(self, frames: torch.Tensor) -> None:
        """Capture run(frames) (fixed input pointer) into a CUDA graph."""
        f = self._check_frames(frames)
        self._graph_input = f
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self._launch(f.data_ptr(), f.stride(0), f.stride(1), None)   # warm-up, attributes
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch(f.data_ptr(), f.stride(0), f.stride(1), None)
        self.graph = g

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.rec

    # --------------------------------------------------------------- results
    def results(self, rec: torch.Tensor | None = None):
        return api._records_to_results(self.rec if rec is None else rec)

    def fits(self, rec: torch.Tensor | None = None):
        return api.records_to_fits(self.rec if rec is None else rec)

    @staticmethod
    def status(rec: torch.Tensor) -> torch.Tensor:
        return rec.view(torch.int32).view(rec.shape[0], 10)[:, 9]


def records_numpy(rec: torch.Tensor) -> np.ndarray:
    """(B,5) float64 records -> structured numpy array (cx, cy, r, score, inliers, status)."""
    r = rec.detach().cpu().numpy()
    dt = np.dtype([("cx", "<f8"), ("cy", "<f8"), ("r", "<f8"), ("score", "<f8"),
                   ("inliers", "<i4"), ("status", "<i4")])
    return r.view(dt).reshape(len(r))
