"""clock64 timeline of the deep cluster variant (k_deep.cu), first cluster: per CTA
and chain warp, mean cycles of each chain segment over samples 16..47.

    python tools/trace_deep.py --config C3 --K 1 --rows 256
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

SEG = ["aready/xfull wait", "z1 + h1 send", "h1full wait", "z2/h2 + z3 partial send", "zfull wait",
       "softmax + delta2 + W3", "fused delta1/W2 + send", "d1full wait + g", "arrive", "-> next sample"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--K", type=int, default=1)
ap.add_argument("--rows", type=int, default=256)
a = ap.parse_args()
c = CONFIGS[a.config]
L = load()
L.pnn_debug_set_trace.argtypes = [ctypes.c_void_p]
C, NCW, TT, PP = 8, 3, 64, 16
buf = torch.zeros(C * NCW * TT * PP, dtype=torch.int64, device="cuda")
X, y = make_split(a.K * a.rows, "train", 0)
net = PNN(c.layers, c.act, c.init, a.K, c.lr)
net.set_kernel("cluster")
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
net.train_epoch(xd, yd)                       # warm (module load, attributes)
torch.cuda.synchronize()
L.pnn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
net.train_epoch(xd, yd)
torch.cuda.synchronize()
L.pnn_debug_set_trace(None)
tr = buf.cpu().numpy().reshape(C, NCW, TT, PP).astype(np.float64)
for cta in range(C):
    for w in range(NCW):
        T = tr[cta, w, 16:48, :10]
        if not T[:, 0].any():
            continue
        per = np.diff(T[:, 0]).mean()
        segs = [np.mean(T[:, i + 1] - T[:, i]) for i in range(9)] + [per - np.mean(T[:, 9] - T[:, 0])]
        print(f"cta {cta} warp {w}: period {per:.0f} | " + " ".join(f"{v:.0f}" for v in segs))
    T = tr[cta, 0, 16:48]
    d = lambda a, b: np.mean(T[:, b] - T[:, a])
    print(f"   seg3: fma {d(3, 10):.0f} reduce {d(10, 11):.0f} act {d(11, 12):.0f} z3part {d(12, 13):.0f} "
          f"send {d(13, 4):.0f}; seg5: z3 sum {d(5, 14):.0f} softmax {d(14, 15):.0f} delta2/W3 {d(15, 6):.0f}")
print("segments:", "; ".join(f"{i}: {s}" for i, s in enumerate(SEG)))
