"""Learned strip scorer: weights container, init and the ECANET01 weight format.

Mirrors the inference half of the reference's ``eca.edgenet``
(/root/reference/pkg/src/eca/edgenet.py:19-47, 86-97, 133-180, 377-449):
same layer shapes (5->8->16->32 valid 3x3 convs + 1x1 head), same
Glorot-uniform init stream (numpy PCG64), same binary weight format.  The
forward pass itself runs only on the GPU (csrc/eca_cnn.cu); training
(edgenet.py:119-130, 213-344) is out of scope for the hot path.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

INPUT_CHANNELS = 5
LAYER_WIDTHS = (8, 16, 32)
EDGE_OFFSET = 3
MAGIC = b"ECANET01"
_SHAPES = [(8, 5, 3, 3), (16, 8, 3, 3), (32, 16, 3, 3), (1, 32, 1, 1)]


class CorruptWeightsError(Exception):
    """Weights stream failed validation (edgenet.py:26-27)."""


@dataclass
class ChannelStats:
    """Per-channel RGB mean / std of the training split (edgenet.py:34-47)."""

    mean: np.ndarray
    std: np.ndarray

    def __post_init__(self) -> None:
        self.mean = np.asarray(self.mean, dtype=np.float64).reshape(3)
        self.std = np.asarray(self.std, dtype=np.float64).reshape(3)
        if not (np.isfinite(self.mean).all() and np.isfinite(self.std).all()):
            raise ValueError("channel stats must be finite")
        if (self.std <= 0).any():
            raise ValueError(f"channel std must be positive, got {self.std}")


def compute_channel_stats(frames) -> ChannelStats:
    """Mean / population std per RGB channel over uint8 frames (edgenet.py:50-64)."""
    n = 0
    s1 = np.zeros(3)
    s2 = np.zeros(3)
    for f in frames:
        d = np.asarray(f, dtype=np.float64).reshape(-1, 3)
        n += d.shape[0]
        s1 += d.sum(axis=0)
        s2 += (d * d).sum(axis=0)
    if n == 0:
        raise ValueError("no frames given")
    mean = s1 / n
    return ChannelStats(mean, np.sqrt(np.maximum(s2 / n - mean * mean, 0.0)))


@dataclass
class ConvLayer:
    kernel: np.ndarray   # (out, in, kh, kw)
    bias: np.ndarray     # (out,)


class EdgeNet:
    """Weights + input normalisation of the strip scorer (edgenet.py:133-180)."""

    def __init__(self, norm: ChannelStats, layers: list[ConvLayer] | None = None, seed: int = 0,
                 dtype=np.float32) -> None:
        self.norm = norm
        self.dtype = np.dtype(dtype)
        if layers is not None:
            self.layers = layers
            self._check()
            return
        rng = np.random.default_rng(seed)
        self.layers = []
        for oc, ic, kh, kw in _SHAPES:       # Glorot uniform, edgenet.py:92-97
            lim = np.sqrt(6.0 / (ic * kh * kw + oc * kh * kw))
            k = rng.uniform(-lim, lim, size=(oc, ic, kh, kw)).astype(self.dtype)
            self.layers.append(ConvLayer(k, np.zeros(oc, dtype=self.dtype)))

    def _check(self) -> None:
        if len(self.layers) != 4:
            raise ValueError(f"expected 4 layers, got {len(self.layers)}")
        want_in = INPUT_CHANNELS
        for i, l in enumerate(self.layers):
            oc, ic, kh, kw = l.kernel.shape
            ks = 1 if i == 3 else 3
            if ic != want_in or kh != ks or kw != ks:
                raise ValueError(f"layer {i} has shape {l.kernel.shape}")
            if l.bias.shape != (oc,):
                raise ValueError(f"layer {i} bias shape {l.bias.shape}")
            want_in = oc
        if self.layers[3].kernel.shape[0] != 1:
            raise ValueError("head must have a single output channel")

    def packed(self) -> np.ndarray:
        """FP32 weights in the layout of ECA_NET_FLOATS (include/eca_b200.h)."""
        self._check()
        if [tuple(l.kernel.shape) for l in self.layers] != _SHAPES:
            raise ValueError("the GPU scorer supports the reference widths 5->8->16->32->1 only")
        parts = []
        for l in self.layers:
            parts.append(np.asarray(l.kernel, dtype=np.float32).ravel())
            parts.append(np.asarray(l.bias, dtype=np.float32).ravel())
        return np.ascontiguousarray(np.concatenate(parts), dtype=np.float32)

    def norm_array(self) -> np.ndarray:
        return np.concatenate([self.norm.mean, self.norm.std]).astype(np.float64)


# ECANET01 stream (edgenet.py:377-437): magic | 6 x f64 channel stats |
# u32 layer count | per layer: 4 x u32 (out, in, kh, kw), f64 kernel, f64 bias.
_STATS = struct.Struct("<6d")
_COUNT = struct.Struct("<I")
_SHAPE = struct.Struct("<4I")


def save_weights(net: EdgeNet) -> bytes:
    """Serialise ``net`` as an ECANET01 stream (edgenet.py:377-387)."""
    blob = bytearray(MAGIC)
    blob += _STATS.pack(*net.norm.mean, *net.norm.std) + _COUNT.pack(len(net.layers))
    for layer in net.layers:
        blob += _SHAPE.pack(*layer.kernel.shape)
        blob += np.asarray(layer.kernel, dtype="<f8").tobytes(order="C")
        blob += np.asarray(layer.bias, dtype="<f8").tobytes(order="C")
    return bytes(blob)


class _Stream:
    """Bounds-checked little-endian cursor over a weights blob."""

    def __init__(self, data: bytes) -> None:
        self.buf, self.pos = memoryview(data), 0

    def bytes(self, n: int) -> memoryview:
        have = len(self.buf) - self.pos
        if n > have:
            raise CorruptWeightsError(
                f"truncated stream: wanted {n} bytes at offset {self.pos}, have {have}")
        self.pos += n
        return self.buf[self.pos - n:self.pos]

    def unpack(self, st: struct.Struct) -> tuple:
        return st.unpack(self.bytes(st.size))

    def f64(self, count: int) -> np.ndarray:
        return np.frombuffer(self.bytes(8 * count), dtype="<f8")


def load_weights(data: bytes, dtype=np.float32) -> EdgeNet:
    """Parse and validate an ECANET01 stream (edgenet.py:390-437); every
    violation raises CorruptWeightsError with the reference's message."""
    rd = _Stream(data)
    if bytes(rd.bytes(len(MAGIC))) != MAGIC:
        raise CorruptWeightsError("bad magic header")
    stats = rd.unpack(_STATS)
    try:
        norm = ChannelStats(np.array(stats[:3]), np.array(stats[3:]))
    except ValueError as exc:
        raise CorruptWeightsError(f"bad channel stats: {exc}") from None
    (count,) = rd.unpack(_COUNT)
    if count != len(_SHAPES):
        raise CorruptWeightsError(f"expected 4 layers, header says {count}")
    layers, chain = [], INPUT_CHANNELS
    for idx, (_, _, want_kh, want_kw) in enumerate(_SHAPES):
        shape = rd.unpack(_SHAPE)
        oc, ic, kh, kw = shape
        if ic != chain:
            raise CorruptWeightsError(f"layer {idx} expects {ic} input channels, chain provides {chain}")
        if (kh, kw) != (want_kh, want_kw) or not 0 < oc <= 4096:
            raise CorruptWeightsError(f"layer {idx} has invalid shape {shape}")
        kernel = rd.f64(oc * ic * kh * kw).reshape(shape)
        bias = rd.f64(oc)
        if not (np.isfinite(kernel).all() and np.isfinite(bias).all()):
            raise CorruptWeightsError(f"layer {idx} contains non-finite weights")
        layers.append(ConvLayer(kernel.astype(dtype), bias.astype(dtype)))
        chain = oc
    if chain != 1:
        raise CorruptWeightsError("head layer must have a single output channel")
    if rd.pos != len(rd.buf):
        raise CorruptWeightsError(f"{len(rd.buf) - rd.pos} trailing bytes after weights")
    return EdgeNet(norm, layers=layers, dtype=dtype)


def save_weights_file(net: EdgeNet, path) -> None:
    from pathlib import Path
    Path(path).write_bytes(save_weights(net))


def load_weights_file(path, dtype=np.float32) -> EdgeNet:
    from pathlib import Path
    return load_weights(Path(path).read_bytes(), dtype=dtype)
