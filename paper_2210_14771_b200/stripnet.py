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


def save_weights(net: EdgeNet) -> bytes:
    """ECANET01 little-endian stream (edgenet.py:377-387)."""
    out = [MAGIC, struct.pack("<6d", *net.norm.mean, *net.norm.std),
           struct.pack("<I", len(net.layers))]
    for l in net.layers:
        out.append(struct.pack("<4I", *l.kernel.shape))
        out.append(np.ascontiguousarray(l.kernel, dtype="<f8").tobytes())
        out.append(np.ascontiguousarray(l.bias, dtype="<f8").tobytes())
    return b"".join(out)


def load_weights(data: bytes, dtype=np.float32) -> EdgeNet:
    """Parse and validate an ECANET01 stream (edgenet.py:390-437)."""
    buf = memoryview(data)
    pos = 0

    def take(n: int) -> memoryview:
        nonlocal pos
        if pos + n > len(buf):
            raise CorruptWeightsError(
                f"truncated stream: wanted {n} bytes at offset {pos}, have {len(buf) - pos}")
        chunk = buf[pos:pos + n]
        pos += n
        return chunk

    if bytes(take(len(MAGIC))) != MAGIC:
        raise CorruptWeightsError("bad magic header")
    st = struct.unpack("<6d", take(48))
    try:
        norm = ChannelStats(np.array(st[:3]), np.array(st[3:]))
    except ValueError as exc:
        raise CorruptWeightsError(f"bad channel stats: {exc}") from None
    (count,) = struct.unpack("<I", take(4))
    if count != 4:
        raise CorruptWeightsError(f"expected 4 layers, header says {count}")
    layers = []
    want_in = INPUT_CHANNELS
    for i in range(count):
        oc, ic, kh, kw = struct.unpack("<4I", take(16))
        ks = 1 if i == 3 else 3
        if ic != want_in:
            raise CorruptWeightsError(f"layer {i} expects {ic} input channels, chain provides {want_in}")
        if kh != ks or kw != ks or oc == 0 or oc > 4096:
            raise CorruptWeightsError(f"layer {i} has invalid shape {(oc, ic, kh, kw)}")
        k = np.frombuffer(take(8 * oc * ic * kh * kw), dtype="<f8").reshape(oc, ic, kh, kw)
        b = np.frombuffer(take(8 * oc), dtype="<f8")
        if not (np.isfinite(k).all() and np.isfinite(b).all()):
            raise CorruptWeightsError(f"layer {i} contains non-finite weights")
        layers.append(ConvLayer(k.astype(dtype), b.astype(dtype)))
        want_in = oc
    if layers[-1].kernel.shape[0] != 1:
        raise CorruptWeightsError("head layer must have a single output channel")
    if pos != len(buf):
        raise CorruptWeightsError(f"{len(buf) - pos} trailing bytes after weights")
    return EdgeNet(norm, layers=layers, dtype=dtype)


def save_weights_file(net: EdgeNet, path) -> None:
    from pathlib import Path
    Path(path).write_bytes(save_weights(net))


def load_weights_file(path, dtype=np.float32) -> EdgeNet:
    from pathlib import Path
    return load_weights(Path(path).read_bytes(), dtype=dtype)
