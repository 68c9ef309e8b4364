"""Small F1 (fp32 mini-batch, 784-256-10, batch 50) run for profiling (tools only)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from datagen import make_rows
from workloads import CONFIGS
from paper_2304_09590_b200 import PNN

c = CONFIGS["F1"]
n = 10 * 50 * 8
X, y = make_rows(0, n, "train", 0)
net = PNN(c.layers, c.act, c.init, 10, c.lr, seed=0)
net.set_minibatch(c.batch)
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
for _ in range(2):
    net.train_epoch(xd, yd)
torch.cuda.synchronize()
print("ok")
