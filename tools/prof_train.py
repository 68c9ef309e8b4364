"""Time (and, under ncu, profile) one training launch of a config shape.

    python tools/prof_train.py --config C4 --K 37 --rows 1024 --kernel auto --reps 3
Prints µs per launch and per-sample latency per CN (CUDA events).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from datagen import make_split  # noqa: E402
from paper_2304_09590_b200 import PNN  # noqa: E402
from workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--K", type=int, default=37)
ap.add_argument("--rows", type=int, default=1024, help="rows per CN")
ap.add_argument("--kernel", default="auto")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
c = CONFIGS[a.config]
X, y = make_split(a.K * a.rows, "train", 0)
net = PNN(c.layers, c.act, c.init, a.K, c.lr)
net.set_kernel(a.kernel)
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
net.train_epoch(xd, yd)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    net.train_epoch(xd, yd)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
us = min(ts)
print(f"{a.config} K={a.K} rows/CN={a.rows} kernel={net.kernel_info()}: {us:.1f} us/launch, "
      f"{us / a.rows * 1e3:.1f} ns/sample/CN, {a.K * a.rows / us:.2f} M samples/s")
