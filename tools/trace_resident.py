"""clock64 timeline of the resident kernel (v7), first two CTAs: per warp and
step t, points 0 loop top, 1 after F(t), 2 after U(t), 3 after the zfull
wait, 4 after finishing sample t-1, 5 after publishing sample t.

    python tools/trace_resident.py --config C4 --K 2 --rows 256
(PNN_RESIDENT_GROUPS=2 selects two CNs per CTA.)
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

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--K", type=int, default=2)
ap.add_argument("--rows", type=int, default=256)
a = ap.parse_args()
c = CONFIGS[a.config]
L = load()
L.pnn_debug_set_trace.argtypes = [ctypes.c_void_p]
NW, TT, PP = 8, 64, 8
buf = torch.zeros(2 * NW * TT * PP, dtype=torch.int64, device="cuda")
X, y = make_split(a.K * a.rows, "train", 0)
net = PNN(c.layers, c.act, c.init, a.K, c.lr)
net.set_kernel("resident")
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
L.pnn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
net.train_epoch(xd, yd)
torch.cuda.synchronize()
L.pnn_debug_set_trace(None)
tr = buf.cpu().numpy().reshape(2, NW, TT, PP).astype(np.float64)
names = ["top", "F", "U", "zwait", "finish(t-1)", "publish(t)"]
for cta in range(2):
    for w in range(NW):
        T = tr[cta, w, 16:48]
        if not T[:, 0].any():
            continue
        per = np.diff(T[:, 0]).mean()
        seg = [(T[:, i + 1] - T[:, i]).mean() for i in range(5)]
        print(f"cta {cta} warp {w}: period {per:.0f} | " +
              " ".join(f"{names[i]}->{names[i+1]} {seg[i]:.0f}" for i in range(5)) +
              f" | publish->next top {np.mean(T[1:, 0] - T[:-1, 5]):.0f}")
base = tr[0, 0, 20, 0]
print("step 20 timeline (cycles from cta0 warp0's step-20 top):")
for cta in range(2):
    for w in range(NW):
        print(f"  cta {cta} w{w}: " + " ".join(f"{tr[cta, w, 20, i] - base:6.0f}" for i in range(6)))
