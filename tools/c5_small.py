"""Small C5 bf16 run for profiling: K=8 CNs, 8*64*R rows, one epoch (tools only)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from datagen import make_rows
from workloads import CONFIGS
from paper_2304_09590_b200 import PNN, PNN_BF16

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS["C5"]
n = 8 * 64 * R
X, y = make_rows(0, n, "train", 0)
net = PNN(c.layers, c.act, c.init, 8, c.lr, seed=0)
net.set_minibatch(64, PNN_BF16)
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
for _ in range(2):
    net.train_epoch(xd, yd)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
net.train_epoch(xd, yd)
b.record()
torch.cuda.synchronize()
print(f"epoch of {R} steps: {a.elapsed_time(b):.3f} ms, {a.elapsed_time(b) / R * 1e3:.1f} us/step")
