"""GPU EdgeNet training against the reference's own outputs
(tests/golden/make_golden_train.py) and the CPU oracle.

Tolerances (FP32 network; the reference's sgemm sums in another order):
logits within 1e-5; loss relative 1e-6; each gradient within 1e-4 of its
layer's largest magnitude; per-epoch losses relative 1e-5; weights after
training within 1e-4; best epoch, early stopping and divergence exact."""

import numpy as np
import pytest

import paper_2210_14771_b200 as eb
from oracle import eca_oracle as orc
from paper_2210_14771_b200 import training as tr

from ._fixtures import load_npz
from .test_oracle_golden import _pack, train_inputs

pytestmark = pytest.mark.gpu


def _net(seed=0):
    return eb.EdgeNet(eb.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=seed)


def _packed_layers(net):
    return _pack([(l.kernel, l.bias) for l in net.layers])


def _grad_close(got, want):
    o = 0
    for oc, ic, kh, kw in [(8, 5, 3, 3), (16, 8, 3, 3), (32, 16, 3, 3), (1, 32, 1, 1)]:
        for n in (oc * ic * kh * kw, oc):
            g, w = got[o:o + n], want[o:o + n]
            assert np.abs(g - w).max() <= 1e-4 * max(np.abs(w).max(), 1e-3), (o, np.abs(g - w).max())
            o += n


def test_forward_and_gradients_match_reference():
    g = load_npz("train.npz")
    net = _net()
    assert np.array_equal(net.packed(), g["w0"])
    x, t = train_inputs()
    logits = tr.forward_logits(net, x[:8])
    assert logits.shape == g["logits"].shape
    assert np.abs(logits - g["logits"]).max() <= 1e-5
    loss, grads = tr.gradients(net, x[:8], t[:8])
    assert loss == pytest.approx(g["loss"][0], rel=1e-6)
    _grad_close(_pack(grads), g["grads"])


@pytest.mark.parametrize("h,w,m", [(7, 9, 3), (9, 130, 5), (11, 300, 2), (7, 1920, 2)])
def test_gradients_match_oracle_shapes(h, w, m):
    """Ragged widths (segments of 128 columns), taller-than-strip inputs
    (train_on_full_frames-style), one full 1080p strip width."""
    rng = np.random.default_rng(h * w + m)
    x = rng.normal(0.0, 1.0, (m, 5, h, w)).astype(np.float32)
    t = rng.uniform(0.0, 1.0, (m, 1, h - 6, w - 6)).astype(np.float32)
    net = _net(seed=h)
    layers = [(l.kernel, l.bias) for l in net.layers]
    want_logits, _ = orc.forward_logits(x, layers)
    assert np.abs(tr.forward_logits(net, x) - want_logits).max() <= 1e-5
    loss, grads = tr.gradients(net, x, t)
    want_loss, want_grads, _ = orc.train_step(x, t, layers, 0.0)
    assert loss == pytest.approx(want_loss, rel=1e-6)
    _grad_close(_pack(grads), _pack(want_grads))


def test_train_loop_matches_reference():
    g = load_npz("train.npz")
    x, t = train_inputs()
    xv, tv = train_inputs(m=10, seed=6)
    net = _net()
    res = tr.train(net, (x, t), (xv, tv), tr.TrainConfig(learning_rate=0.05, batch_size=4, max_epochs=6,
                                                          early_stop_patience=2), seed=3)
    assert res.best_epoch == g["best_epoch"][0]
    assert np.allclose(res.train_losses, g["train_losses"], rtol=1e-5, atol=0)
    assert np.allclose(res.val_losses, g["val_losses"], rtol=1e-5, atol=0)
    assert np.abs(_packed_layers(net) - g["w_trained"]).max() <= 1e-4
    net = _net()
    res = tr.train(net, (x, t), None, tr.TrainConfig(learning_rate=0.02, batch_size=5, max_epochs=2,
                                                      shuffle=False))
    assert np.allclose(res.train_losses, g["train_losses_noval"], rtol=1e-5, atol=0)
    assert np.abs(_packed_layers(net) - g["w_noval"]).max() <= 1e-4


def test_early_stopping_matches_oracle():
    x, t = train_inputs(m=16, w=40, seed=9)
    xv, tv = train_inputs(m=6, w=40, seed=10)
    net = _net(seed=4)
    layers = [(l.kernel.copy(), l.bias.copy()) for l in net.layers]
    res = tr.train(net, (x, t), (xv, tv), tr.TrainConfig(learning_rate=3.0, batch_size=4, max_epochs=12,
                                                          early_stop_patience=2), seed=1)
    best, tl, vl, be = orc.train(layers, x, t, xv, tv, lr=3.0, batch=4, patience=2, epochs=12, seed=1)
    assert res.best_epoch == be and len(res.val_losses) == len(vl)
    assert np.allclose(res.val_losses, vl, rtol=1e-4, atol=0)


def test_divergence_raises_like_reference():
    x, t = train_inputs(m=12, w=20, seed=2)
    net = _net()
    layers = [(l.kernel.copy(), l.bias.copy()) for l in net.layers]
    with pytest.raises(FloatingPointError) as want:
        orc.train(layers, x, t, None, None, lr=1e30, batch=4, epochs=3, seed=0)
    with pytest.raises(tr.TrainingDivergedError) as got:
        tr.train(net, (x, t), None, tr.TrainConfig(learning_rate=1e30, batch_size=4, max_epochs=3), seed=0)
    assert str(got.value) == str(want.value)


def test_training_rejects_bad_input():
    net = _net()
    with pytest.raises(ValueError, match="training set is empty"):
        tr.train(net, (np.zeros((0, 5, 7, 20), np.float32), np.zeros((0, 1, 1, 14), np.float32)), None)
    with pytest.raises(ValueError, match="receptive field"):
        tr.forward_logits(net, np.zeros((1, 5, 6, 20), np.float32))


def test_gradients_many_tiles_per_cta():
    """64 strips x 1920: every persistent conv CTA loops over several tiles
    and every weight-gradient CTA over several 32-column units (ragged row
    ends included), against the oracle.  Inputs, weights and biases are
    non-negative / positive so no pre-activation is near 0: at this size a
    value within FP32 rounding of 0 can get different ReLU masks on the two
    sides (a near-tie: one flipped unit moves a gradient element by a whole
    term, K7); this test is about the tiling, not ties."""
    from paper_2210_14771_b200.stripnet import ConvLayer

    rng = np.random.default_rng(17)
    x = np.abs(rng.normal(0.0, 1.0, (64, 5, 7, 1920))).astype(np.float32)
    t = rng.uniform(0.0, 1.0, (64, 1, 1, 1914)).astype(np.float32)
    net = _net(seed=5)
    net.layers = [ConvLayer(np.abs(l.kernel), np.full_like(l.bias, 0.1)) if i < 3 else l
                  for i, l in enumerate(net.layers)]
    layers = [(l.kernel, l.bias) for l in net.layers]
    want_logits, _ = orc.forward_logits(x, layers)
    assert np.abs(tr.forward_logits(net, x) - want_logits).max() <= 1e-5 * max(1.0, np.abs(want_logits).max())
    loss, grads = tr.gradients(net, x, t)
    want_loss, want_grads, _ = orc.train_step(x, t, layers, 0.0)
    assert loss == pytest.approx(want_loss, rel=1e-6)
    _grad_close(_pack(grads), _pack(want_grads))


def test_concurrent_streams_match_sequential():
    """Two trainers stepping on two streams at once (their tensor-core CTAs
    share SMs: the shared-memory padding must keep their TMEM allocations
    within 512 columns per SM) give the results of running them one after
    the other."""
    import torch

    rng = np.random.default_rng(23)
    dev = torch.device("cuda", 0)
    xs = [torch.from_numpy(rng.normal(0.0, 1.0, (16, 5, 7, 1920)).astype(np.float32)).to(dev) for _ in range(2)]
    ts = [torch.from_numpy(rng.uniform(0.0, 1.0, (16, 1, 1, 1914)).astype(np.float32)).to(dev) for _ in range(2)]

    def run(concurrent: bool):
        trainers = [tr._Trainer(_net(seed=k), 7, 1920, 16, dev) for k in range(2)]
        losses = [torch.zeros(8, dtype=torch.float64, device=dev) for _ in range(2)]
        streams = [torch.cuda.Stream(dev) for _ in range(2)]
        torch.cuda.synchronize()
        for step in range(8):
            for k in range(2):
                with torch.cuda.stream(streams[k] if concurrent else streams[0]):
                    trainers[k].forward(xs[k], None, 16)
                    trainers[k].backward(xs[k], ts[k], None, 16, losses[k][step:step + 1])
                    trainers[k].sgd(0.05)
        torch.cuda.synchronize()
        return [t.weights.cpu().numpy() for t in trainers], [l.cpu().numpy() for l in losses]

    w_seq, l_seq = run(False)
    w_con, l_con = run(True)
    for a, b in zip(w_seq + l_seq, w_con + l_con):
        assert np.array_equal(a, b)
