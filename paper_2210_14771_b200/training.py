"""Learned-variant training on the GPU.

Drop-in for the training half of ``eca.edgenet`` (edgenet.py:119-130,
182-225, 236-344): ``forward_logits``, ``gradients`` (the reference's
``EdgeNet.backward`` after the BCE), ``train`` with ``TrainConfig`` /
``TrainResult`` / ``TrainingDivergedError``.  Forward, backward and the SGD
update are hand-written kernels in libeca_b200.so (csrc/eca_train.cu); the
epoch loop stays on the host like the reference's, but a whole epoch is
enqueued without synchronising: per-step losses stay on the device, a
device flag turns the remaining SGD updates into no-ops after a non-finite
loss (the reference raises before that update), and the host reads the
losses once per epoch (early stopping needs the validation loss).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .api import _device, _ptr, _stream
from .stripnet import _SHAPES, ConvLayer, EdgeNet

NET_FLOATS = _lib.NET_FLOATS


class TrainingDivergedError(Exception):
    """A training step produced a non-finite loss (edgenet.py:29-30)."""


@dataclass(frozen=True)
class TrainConfig:
    """edgenet.py:244-254 (defaults follow the published recipe)."""
    learning_rate: float = 0.001
    batch_size: int = 8
    target_blur_sigma: float = 3.0
    early_stop_patience: int = 5
    max_epochs: int = 50
    shuffle: bool = True
    train_on_full_frames: bool = False


@dataclass
class TrainResult:
    net: EdgeNet
    train_losses: list[float] = field(default_factory=list)
    val_losses: list[float] = field(default_factory=list)
    best_epoch: int = -1


def unpack(weights: np.ndarray, dtype=np.float32) -> list[ConvLayer]:
    """ECA_NET_FLOATS packed weights -> reference-shaped layers."""
    w = np.asarray(weights, dtype=np.float32).ravel()
    if w.size != NET_FLOATS:
        raise ValueError(f"expected {NET_FLOATS} packed weights, got {w.size}")
    out, o = [], 0
    for oc, ic, kh, kw in _SHAPES:
        n = oc * ic * kh * kw
        k = w[o:o + n].reshape(oc, ic, kh, kw).astype(dtype)
        b = w[o + n:o + n + oc].astype(dtype)
        out.append(ConvLayer(k, b))
        o += n + oc
    return out


def _samples(x, dev) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    t = t.to(dev, dtype=torch.float32).contiguous()
    if t.ndim != 4:
        raise ValueError(f"expected a (B, C, h, W) array, got shape {tuple(t.shape)}")
    return t


class _Trainer:
    """Device state of one network: packed weights, workspace, buffers."""

    def __init__(self, net: EdgeNet, h: int, w: int, m_max: int, dev):
        self.dev, self.h, self.w = dev, h, w
        self.lib = _lib.load()
        self.weights = torch.from_numpy(net.packed()).to(dev)
        self.grads = torch.zeros(NET_FLOATS, dtype=torch.float32, device=dev)
        nb = ctypes.c_int64()
        _lib.check(self.lib.eca_train_workspace_bytes(m_max, h, w, ctypes.byref(nb)),
                   "eca_train_workspace_bytes")
        self.ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
        self.ws_bytes = nb.value
        self.diverged = torch.zeros(1, dtype=torch.int32, device=dev)

    @property
    def st(self):   # the current stream at call time (a CUDA-graph capture stream inside one)
        return _stream(self.dev)

    def forward(self, x: torch.Tensor, idx, m: int, logits: torch.Tensor | None = None) -> None:
        _lib.check(self.lib.eca_edgenet_forward(
            _ptr(x), idx, m, self.h, self.w, _ptr(self.weights), _ptr(self.ws), self.ws_bytes,
            None if logits is None else _ptr(logits), self.st), "eca_edgenet_forward")

    def backward(self, x, t, idx, m: int, loss_slot: torch.Tensor, grads: bool = True) -> None:
        _lib.check(self.lib.eca_edgenet_backward(
            _ptr(x), _ptr(t), idx, m, self.h, self.w, _ptr(self.weights), _ptr(self.ws), self.ws_bytes,
            _ptr(self.grads) if grads else None, _ptr(loss_slot), _ptr(self.diverged), self.st),
            "eca_edgenet_backward")

    def sgd(self, lr: float) -> None:
        _lib.check(self.lib.eca_sgd_step(_ptr(self.weights), _ptr(self.grads), ctypes.c_float(lr),
                                          _ptr(self.diverged), self.st), "eca_sgd_step")


def _check_input(x: torch.Tensor) -> None:
    if x.shape[1] != 5:
        raise ValueError(f"expected input of shape (B, 5, h, W), got {tuple(x.shape)}")
    if x.shape[2] < 7 or x.shape[3] < 7:
        raise ValueError(f"input spatial size {x.shape[2]}x{x.shape[3]} is below the 7x7 receptive field")


def forward_logits(net: EdgeNet, x, device=None) -> np.ndarray:
    """Pre-sigmoid activations (B, 1, h-6, W-6) of a (B, 5, h, W) batch
    (edgenet.py:182-205) on the GPU."""
    dev = _device(device)
    xd = _samples(x, dev)
    _check_input(xd)
    m, _, h, w = xd.shape
    tr = _Trainer(net, h, w, m, dev)
    out = torch.empty((m, 1, h - 6, w - 6), dtype=torch.float32, device=dev)
    tr.forward(xd, None, m, out)
    return out.cpu().numpy()


def gradients(net: EdgeNet, x, targets, device=None):
    """(loss, per-layer (dkernel, dbias)) of one batch: the reference's
    forward_logits + _bce_with_logits + backward(dlogits) (edgenet.py:306-316)."""
    dev = _device(device)
    xd, td = _samples(x, dev), _samples(targets, dev)
    _check_input(xd)
    m, _, h, w = xd.shape
    tr = _Trainer(net, h, w, m, dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    tr.forward(xd, None, m)
    tr.backward(xd, td, None, m, loss)
    g = unpack(tr.grads.cpu().numpy())
    return float(loss.item()), [(l.kernel, l.bias) for l in g]


def train(net: EdgeNet, train_samples, val_samples, cfg: TrainConfig | None = None, seed: int = 0,
          device=None) -> TrainResult:
    """Plain SGD on soft BCE against blurred edge-map targets, validation-loss
    early stopping, best-validation snapshot (edgenet.py:277-344), on the GPU."""
    cfg = cfg or TrainConfig()
    dev = _device(device)
    xs, ts = _samples(train_samples[0], dev), _samples(train_samples[1], dev)
    if len(xs) == 0:
        raise ValueError("training set is empty")
    _check_input(xs)
    if val_samples is not None:
        vx, vt = _samples(val_samples[0], dev), _samples(val_samples[1], dev)
    n, _, h, w = xs.shape
    vb = max(cfg.batch_size, 32)
    tr = _Trainer(net, h, w, max(cfg.batch_size, vb if val_samples is not None else 1), dev)
    plane = (h - 6) * (w - 6)
    result = TrainResult(net)
    rng = np.random.default_rng(seed)
    best = tr.weights.clone()
    best_val = np.inf
    stale = 0
    steps = list(range(0, n, cfg.batch_size))
    losses = torch.zeros(len(steps), dtype=torch.float64, device=dev)
    vsteps = list(range(0, len(vx), vb)) if val_samples is not None else []
    vlosses = torch.zeros(max(1, len(vsteps)), dtype=torch.float64, device=dev)
    order_d = torch.empty(n, dtype=torch.int32, device=dev)

    def epoch_steps():
        for k, s in enumerate(steps):
            m = min(cfg.batch_size, n - s)
            idx = ctypes.c_void_p(order_d.data_ptr() + 4 * s)
            tr.forward(xs, idx, m)
            tr.backward(xs, ts, idx, m, losses[k:k + 1])
            if cfg.learning_rate != 0.0:
                tr.sgd(cfg.learning_rate)

    # An epoch's launch sequence depends only on (n, batch size): from the
    # second epoch on it replays as one CUDA graph (the permutation is copied
    # into order_d in front of it), instead of ~16 launches per step from the
    # host.  The first epoch runs eagerly (and warms the kernels up).
    graph = None
    for epoch in range(cfg.max_epochs):
        order = rng.permutation(n) if cfg.shuffle else np.arange(n)
        order_d.copy_(torch.from_numpy(order.astype(np.int32)))
        if graph is not None:
            graph.replay()
        elif epoch == 0 or len(steps) < 4:
            epoch_steps()
        else:
            torch.cuda.synchronize(dev)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                epoch_steps()
            graph.replay()
        lh = losses.cpu().numpy()
        bad = np.flatnonzero(~np.isfinite(lh))
        if len(bad):
            net.layers = unpack(tr.weights.cpu().numpy(), net.dtype)
            raise TrainingDivergedError(
                f"non-finite loss at epoch {epoch}, sample offset {steps[bad[0]]}")
        total, count = 0.0, 0
        for k, s in enumerate(steps):
            size = min(cfg.batch_size, n - s) * plane
            total += float(lh[k]) * size
            count += size
        result.train_losses.append(total / count)
        if val_samples is not None:
            for k, s in enumerate(vsteps):
                m = min(vb, len(vx) - s)
                xv = vx[s:s + m]
                tr.forward(xv, None, m)
                tr.backward(xv, vt[s:s + m], None, m, vlosses[k:k + 1], grads=False)
            vh = vlosses.cpu().numpy()
            total, count = 0.0, 0
            for k, s in enumerate(vsteps):
                size = min(vb, len(vx) - s) * plane
                total += float(vh[k]) * size
                count += size
            val_loss = total / max(count, 1)
            result.val_losses.append(val_loss)
            if val_loss < best_val:
                best_val = val_loss
                best = tr.weights.clone()
                result.best_epoch = epoch
                stale = 0
            else:
                stale += 1
                if stale >= cfg.early_stop_patience:
                    break
        else:
            best = tr.weights.clone()
            result.best_epoch = epoch
    net.layers = unpack(best.cpu().numpy(), net.dtype)
    return result
