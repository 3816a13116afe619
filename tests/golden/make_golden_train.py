"""Golden fixtures for GPU EdgeNet training, made by running the
REFERENCE's edgenet module (forward_logits / backward / _bce_with_logits /
train, /root/reference/pkg/src/eca/edgenet.py) in the build container:

    python tests/golden/make_golden_train.py

Inputs are regenerated from seeds by the tests (train_inputs below is
copied there), so only the reference's outputs are stored (train.npz).
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from eca import edgenet as en  # noqa: E402

OUT = Path(__file__).resolve().parent


def train_inputs(m=24, h=7, w=64, seed=5):
    """Synthetic RGBXY strips and soft targets (same recipe in the tests)."""
    rng = np.random.default_rng(seed)
    x = rng.normal(0.0, 1.0, (m, 5, h, w)).astype(np.float32)
    t = rng.uniform(0.0, 1.0, (m, 1, h - 6, w - 6)).astype(np.float32)
    return x, t


def packed(layers):
    return np.concatenate([np.concatenate([l.kernel.ravel(), l.bias.ravel()]) for l in layers]).astype(np.float32)


def main():
    out = {}
    net = en.EdgeNet(en.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=0)
    out["w0"] = packed(net.layers)
    x, t = train_inputs()
    # one batch: logits, loss, gradients (edgenet.py:182-225, 236-241, 313-316)
    xb, tb = x[:8], t[:8]
    logits, caches = net.forward_logits(xb, keep_caches=True)
    out["logits"] = logits
    out["loss"] = np.array([en._bce_with_logits(logits, tb)])
    dlog = (en._sigmoid(logits) - tb.astype(logits.dtype)) / logits.size
    grads = net.backward(dlog, caches)
    out["grads"] = np.concatenate([np.concatenate([dk.ravel(), db.ravel()]) for dk, db in grads]).astype(np.float32)
    # a short training run with validation + early stopping (edgenet.py:277-344)
    xv, tv = train_inputs(m=10, seed=6)
    cfg = en.TrainConfig(learning_rate=0.05, batch_size=4, max_epochs=6, early_stop_patience=2)
    net2 = en.EdgeNet(en.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=0)
    res = en.train(net2, (x, t), (xv, tv), cfg, seed=3)
    out["train_losses"] = np.array(res.train_losses)
    out["val_losses"] = np.array(res.val_losses)
    out["best_epoch"] = np.array([res.best_epoch])
    out["w_trained"] = packed(net2.layers)
    # no validation set: the last epoch's weights
    net3 = en.EdgeNet(en.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=0)
    res3 = en.train(net3, (x, t), None, en.TrainConfig(learning_rate=0.02, batch_size=5, max_epochs=2,
                                                        shuffle=False), seed=0)
    out["train_losses_noval"] = np.array(res3.train_losses)
    out["w_noval"] = packed(net3.layers)
    np.savez_compressed(OUT / "train.npz", **out)
    print({k: v.shape for k, v in out.items()}, res.train_losses, res.val_losses, res.best_epoch)


if __name__ == "__main__":
    main()
