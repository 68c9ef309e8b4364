"""Small C4 run on the resident kernel for profiling (tools only): K CNs x rows."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from datagen import make_rows
from workloads import CONFIGS
from paper_2304_09590_b200 import PNN

c = CONFIGS["C4"]
K = int(sys.argv[1]) if len(sys.argv) > 1 else 148
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 256
X, y = make_rows(0, K * rows, "train", 0)
net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
net.set_kernel("resident")
if len(sys.argv) > 3:
    net.set_variant(sys.argv[3])
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
net.train_epoch(xd, yd)
torch.cuda.synchronize()
print("ok")
