"""Small C3 run on the cluster kernel for profiling (tools only)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from datagen import make_rows
from workloads import CONFIGS
from paper_2304_09590_b200 import PNN

c = CONFIGS["C3"]
K = 16
X, y = make_rows(0, K * 400, "train", 0)
net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
net.set_kernel("cluster")
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
net.train_epoch(xd, yd)
torch.cuda.synchronize()
print("ok")
