"""clock64 timeline of the TMEM resident variant (v11, k_tmem.cu), first two CTAs.
Per warp and step s, points: 0 loop top, 1 after the x(s) wait, 2 F(s) done,
3 chain (s-1) after its aready wait, 4 after z1/h, 5 after the pair's logit exchange,
6 chain done (gready arrived), 7 Gram record of the pair's next sample done,
8 U(s) after its gready wait, 9 U(s) done.

    python tools/trace_tmem.py --K 1 --rows 256
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
ap.add_argument("--K", type=int, default=1)
ap.add_argument("--rows", type=int, default=256)
a = ap.parse_args()
c = CONFIGS["C4"]
L = load()
L.pnn_debug_set_trace.argtypes = [ctypes.c_void_p]
NW, TT, PP = 8, 64, 16
buf = torch.zeros(2 * NW * TT * PP, dtype=torch.int64, device="cuda")
X, y = make_split(a.K * a.rows, "train", 0)
net = PNN(c.layers, c.act, c.init, a.K, c.lr)
net.set_variant("tmem")
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
net.train_epoch(xd, yd)          # warm (module load)
L.pnn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
net.train_epoch(xd, yd)
torch.cuda.synchronize()
L.pnn_debug_set_trace(None)
tr = buf.cpu().numpy().reshape(2, NW, TT, PP).astype(np.float64)
S0, S1 = 16, 56
for w in range(NW):
    T = tr[0, w, S0:S1]
    per = np.diff(T[:, 0]).mean()
    xw = (T[:, 1] - T[:, 0]).mean()
    f = (T[:, 2] - T[:, 1]).mean()
    uw = (T[:, 8] - np.maximum(T[:, 2], T[:, 7])).mean()
    u = (T[:, 9] - T[:, 8]).mean()
    ch = T[T[:, 3] > 0]
    s = f"warp {w}: period {per:.0f} | xwait {xw:.0f} F {f:.0f} gwait {uw:.0f} U {u:.0f}"
    if len(ch):
        d = lambda i, j: np.mean(ch[:, j] - ch[:, i])
        s += (f" | chain: await {np.mean(ch[:, 3] - ch[:, 2]):.0f} z/h {d(3, 4):.0f} logits+bar {d(4, 5):.0f}"
              f" softmax..arrive {d(5, 6):.0f} gram {d(6, 7):.0f}")
    print(s)
done = []
for s in range(S0, S1):
    w = 2 * ((s - 1) & 3)
    if tr[0, w, s, 6] > 0:
        done.append(tr[0, w, s, 6])
print(f"chain period (cta 0): {np.diff(done).mean():.0f} cycles/sample")
t0 = tr[0, 0, 20, 0]
print("timeline (cycles rel. to warp 0 step 20 top): step s: [warp: top F-end U-start U-end] chain(s-1) on pair (s-1)&3: start end")
for s in range(20, 28):
    row = " ".join(f"w{w}:{tr[0, w, s, 0] - t0:6.0f}/{tr[0, w, s, 2] - t0:6.0f}/{tr[0, w, s, 8] - t0:6.0f}/{tr[0, w, s, 9] - t0:6.0f}" for w in range(NW))
    w = 2 * ((s - 1) & 3)
    print(f"s={s}: {row} | chain {tr[0, w, s, 3] - t0:6.0f}..{tr[0, w, s, 6] - t0:6.0f} gram..{tr[0, w, s, 7] - t0:6.0f}")
