"""clock64 timeline of the paired v8 resident kernel, CTA 0 (tools only).  Per warp and step p
(2 samples): F pass, the chain it runs (if any: samples 2p-2 / 2p-1 on pairs (c & 3)), U pass.
Points: 0 top, 1 after F, 3 chain after its aready wait, 6 chain done, 12 before U, 2 after U.

    python tools/trace_v8p.py --K 74 --rows 256
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
ap.add_argument("--K", type=int, default=74)
ap.add_argument("--rows", type=int, default=256)
a = ap.parse_args()
c = CONFIGS["C4"]
L = load()
L.pnn_debug_set_trace.argtypes = [ctypes.c_void_p]
NW, TT, PP = 8, 64, 16
buf = torch.zeros(2 * NW * TT * PP, dtype=torch.int64, device="cuda")
X, y = make_split(a.K * a.rows, "train", 0)
net = PNN(c.layers, c.act, c.init, a.K, c.lr)
net.set_variant("v8")
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
net.train_epoch(xd, yd)
L.pnn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
net.train_epoch(xd, yd)
torch.cuda.synchronize()
L.pnn_debug_set_trace(None)
tr = buf.cpu().numpy().reshape(2, NW, TT, PP).astype(np.float64)
steps = range(20, 30, 2)      # s = 2p (even rows hold step p)
t0 = tr[0, 0, 20, 0]
for s in steps:
    line = []
    for w in range(NW):
        T = tr[0, w, s] - t0
        ch = f" C[{T[3]:.0f},{T[6]:.0f}]" if tr[0, w, s, 3] > 0 else ""
        line.append(f"w{w}: F[{T[0]:.0f},{T[1]:.0f}]{ch} U[{T[12]:.0f},{T[2]:.0f}]")
    print(f"p={s // 2}:")
    for l in line:
        print("   ", l)
per = []
for w in range(NW):
    T = tr[0, w, 16:48:2]
    per.append(np.diff(T[:, 0]).mean())
    f = np.mean(T[:, 1] - T[:, 0]); u = np.mean(T[:, 2] - T[:, 12])
    chm = T[T[:, 3] > 0]
    chd = np.mean(chm[:, 6] - chm[:, 3]) if len(chm) else 0
    print(f"warp {w}: step {per[-1]:.0f} cycles (2 samples) | F {f:.0f} U {u:.0f} chain {chd:.0f} (x{len(chm)})")
# chain segments (mean over the chains of CTA 0 in steps 8..31)
seg = [(3, 7, "z1/h"), (7, 8, "logits+reduce"), (8, 9, "publish"), (9, 5, "exchange wait"),
       (5, 10, "z2+softmax"), (10, 11, "delta1/g"), (11, 6, "updates/arrive")]
rows = []
for w in range(NW):
    for s in range(16, 64, 2):
        T = tr[0, w, s]
        if T[3] > 0 and T[6] > 0:
            rows.append(T)
rows = np.array(rows)
print("chain segments (cycles):", " | ".join(f"{n} {np.mean(rows[:, b] - rows[:, a]):.0f}" for a, b, n in seg),
      f"| total {np.mean(rows[:, 6] - rows[:, 3]):.0f}")
