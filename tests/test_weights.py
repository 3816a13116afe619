"""ECANET01 weights stream: save / load round trip and
the CorruptWeightsError contract, mirroring the reference's own tests
(/root/reference/pkg/tests/test_edgenet.py:247-279), plus byte equality with
the blob the reference wrote for the golden net (tests/golden/learned.npz)."""

import numpy as np
import pytest

import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import stripnet

from ._fixtures import load_npz

NORM = eb.ChannelStats([100.0] * 3, [50.0] * 3)


def test_save_matches_reference_blob():
    blob = load_npz("learned.npz")["blob"].tobytes()
    assert eb.save_weights(eb.EdgeNet(NORM, seed=0)) == blob


def test_load_reference_blob():
    blob = load_npz("learned.npz")["blob"].tobytes()
    net = eb.load_weights(blob)
    ref = load_npz("learned.npz")
    for i, layer in enumerate(net.layers):
        assert layer.kernel.dtype == np.float32
        assert np.array_equal(layer.kernel, ref[f"w{i}"].astype(np.float32))
        assert np.array_equal(layer.bias, ref[f"b{i}"].astype(np.float32))
    assert np.array_equal(net.packed(), eb.EdgeNet(NORM, seed=0).packed())


def test_weights_roundtrip_bit_identical():
    net = eb.EdgeNet(NORM, seed=8, dtype=np.float64)
    clone = eb.load_weights(eb.save_weights(net), dtype=np.float64)
    for a, b in zip(net.layers, clone.layers):
        assert np.array_equal(a.kernel, b.kernel) and np.array_equal(a.bias, b.bias)
    assert np.array_equal(clone.norm.mean, net.norm.mean)
    assert np.array_equal(clone.norm.std, net.norm.std)


def test_weights_file_roundtrip(tmp_path):
    net = eb.EdgeNet(NORM, seed=3)
    path = tmp_path / "net.ecanet"
    stripnet.save_weights_file(net, path)
    assert np.array_equal(stripnet.load_weights_file(path).packed(), net.packed())


def test_weights_truncated_stream_rejected():
    blob = eb.save_weights(eb.EdgeNet(NORM, seed=9))
    with pytest.raises(eb.CorruptWeightsError, match="truncated stream"):
        eb.load_weights(blob[: len(blob) // 2])
    for cut in (0, 4, 8, 40, 56, 60, 75):
        with pytest.raises(eb.CorruptWeightsError):
            eb.load_weights(blob[:cut])


def test_weights_bad_magic_rejected():
    blob = eb.save_weights(eb.EdgeNet(NORM, seed=9))
    with pytest.raises(eb.CorruptWeightsError, match="bad magic header"):
        eb.load_weights(b"NOTMAGIC" + blob[8:])


def test_weights_wrong_channel_count_rejected():
    net = eb.EdgeNet(NORM, seed=9)
    net.layers[0].kernel = np.zeros((8, 4, 3, 3))   # 4 input channels instead of 5
    with pytest.raises(eb.CorruptWeightsError, match="layer 0 expects 4 input channels"):
        eb.load_weights(eb.save_weights(net))


def test_weights_trailing_bytes_rejected():
    blob = eb.save_weights(eb.EdgeNet(NORM, seed=9))
    with pytest.raises(eb.CorruptWeightsError, match="1 trailing bytes"):
        eb.load_weights(blob + b"\x00")


def test_weights_bad_stats_layers_and_values_rejected():
    import struct
    blob = bytearray(eb.save_weights(eb.EdgeNet(NORM, seed=9)))
    bad_std = blob.copy()
    bad_std[8 + 24:8 + 32] = struct.pack("<d", 0.0)
    with pytest.raises(eb.CorruptWeightsError, match="bad channel stats"):
        eb.load_weights(bytes(bad_std))
    bad_count = blob.copy()
    bad_count[56:60] = struct.pack("<I", 3)
    with pytest.raises(eb.CorruptWeightsError, match="expected 4 layers"):
        eb.load_weights(bytes(bad_count))
    bad_kernel = blob.copy()
    bad_kernel[60 + 16:60 + 24] = struct.pack("<d", float("nan"))
    with pytest.raises(eb.CorruptWeightsError, match="non-finite"):
        eb.load_weights(bytes(bad_kernel))
    bad_shape = blob.copy()
    bad_shape[60 + 8:60 + 12] = struct.pack("<I", 5)   # layer 0 kh = 5
    with pytest.raises(eb.CorruptWeightsError, match="invalid shape"):
        eb.load_weights(bytes(bad_shape))
