"""clock64 timeline of the resident mini-batch kernel (k_mbres.cu), CTA 0: per warp,
mean cycles of each phase over steps 2..15.

    python tools/trace_mbres.py [--K 10] [--rows-per-cn 1000]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from datagen import make_split  # noqa: E402
from paper_2304_09590_b200 import PNN, load  # noqa: E402
from workloads import CONFIGS  # noqa: E402

SEG = ["P1 forward rows", "P1 barrier", "P2 partial logits + send", "zfull wait", "P3 softmax/delta2",
       "P3 barrier", "P4 delta1 + barrier + W2/b updates", "P5 W1 update rows", "end barrier"]
ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=10)
ap.add_argument("--rows-per-cn", type=int, default=1000)
a = ap.parse_args()
c = CONFIGS["F1"]
L = load()
L.pnn_debug_set_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(8 * 16 * 16, dtype=torch.int64, device="cuda")
X, y = make_split(a.K * a.rows_per_cn, "train", 0)
net = PNN(c.layers, c.act, c.init, a.K, c.lr)
net.set_minibatch(c.batch)
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
net.train_epoch(xd, yd)
torch.cuda.synchronize()
L.pnn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
net.train_epoch(xd, yd)
torch.cuda.synchronize()
L.pnn_debug_set_trace(None)
tr = buf.cpu().numpy().reshape(8, 16, 16).astype(np.float64)
for w in range(8):
    T = tr[w, 2:16, :10]
    per = np.diff(T[:, 0]).mean()
    print(f"warp {w}: step {per:.0f} | " + " ".join(f"{np.mean(T[:, i + 1] - T[:, i]):.0f}" for i in range(9)))
print("segments:", "; ".join(f"{i}: {s}" for i, s in enumerate(SEG)))
