"""ncu target: a few EdgeNet SGD steps (batch 8 strips of 5x7x1920)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2210_14771_b200 as eb
from paper_2210_14771_b200 import training as tr
rng = np.random.default_rng(0)
x = rng.normal(0, 1, (32, 5, 7, 1920)).astype(np.float32)
t = rng.uniform(0, 1, (32, 1, 1, 1914)).astype(np.float32)
net = eb.EdgeNet(eb.ChannelStats((100.0,) * 3, (50.0,) * 3), seed=0)
tr.train(net, (x, t), None, tr.TrainConfig(learning_rate=0.001, batch_size=8, max_epochs=1))
torch.cuda.synchronize()
print("ok")
