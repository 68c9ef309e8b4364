"""clock64 timeline of the resident kernel (v8), first two CTAs: per warp and
step s, points 0 loop top, 1 after F(s), 2 after U(s); for the warp that runs
the chain of sample s-1: 3 after its waits (row sums, previous chain), 4 after
publishing its partial logits, 5 after the exchange wait, 6 chain done.

    python tools/trace_resident.py --config C4 --K 1 --rows 256
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
ap.add_argument("--K", type=int, default=1)
ap.add_argument("--rows", type=int, default=256)
a = ap.parse_args()
c = CONFIGS[a.config]
L = load()
L.pnn_debug_set_trace.argtypes = [ctypes.c_void_p]
NW, TT, PP = 8, 64, 16
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
for cta in range(2):
    for w in range(NW):
        T = tr[cta, w, 16:48]
        if not T[:, 0].any():
            continue
        per = np.diff(T[:, 0]).mean()
        f, u = (T[:, 1] - T[:, 0]).mean(), (T[:, 2] - T[:, 1]).mean()
        ch = T[T[:, 3] > 0]
        cs = ""
        if len(ch):
            cs = (f" | chain: wait {np.mean(ch[:, 3] - ch[:, 2]):.0f} publish {np.mean(ch[:, 4] - ch[:, 3]):.0f}"
                  f" xwait {0:.0f} exch {np.mean(ch[:, 5] - ch[:, 4]):.0f} finish {np.mean(ch[:, 6] - ch[:, 5]):.0f}")
        if len(ch):
            d = lambda a, b: np.mean(ch[:, b] - ch[:, a])
            cs += (f"\n      publish = z1/h {d(3, 7):.0f} + W2/logits/reduce {d(7, 8):.0f} + store/st.async/arrive "
                   f"{d(8, 9):.0f} + x issue/wait {d(9, 4):.0f}; finish = softmax {d(5, 10):.0f} + delta1/g "
                   f"{d(10, 11):.0f} + updates/arrive {d(11, 6):.0f}")
        print(f"cta {cta} warp {w}: period {per:.0f} | F {f:.0f} U {u:.0f}{cs}")
# chain period: time between consecutive chain completions (point 6 of the owning warp)
done = []
for s in range(17, 48):
    w = (s - 1) % NW
    if tr[0, w, s, 6] > 0:
        done.append(tr[0, w, s, 6])
if len(done) > 2:
    print(f"chain period (cta 0): {np.diff(done).mean():.0f} cycles/sample")
print("per-sample chain timeline, cta 0 (cycles rel. to first): c, pair warps: [TR2 (ready to start), TR3 (waits done), TR4, TR5, TR6] for warp A | B")
rows = []
for cc in range(20, 30):
    s = cc + 1
    wa = 2 * (cc & 3)
    rows.append((cc, [tr[0, wa, s, i] for i in (2, 3, 4, 5, 6)], [tr[0, wa + 1, s, i] for i in (2, 3, 4, 5, 6)]))
t0 = rows[0][1][1]
for cc, A, B in rows:
    print(f"  c={cc}: A " + " ".join(f"{v - t0:7.0f}" for v in A) + " | B " + " ".join(f"{v - t0:7.0f}" for v in B))
