"""clock64 timeline of the resident kernel's tail warp and pass warp 0 (CTA 0).

    python tools/trace_resident.py --config C4 --K 1 --rows 256
Tail points: 0 loop top, 1 acc ready, 2 logits reduced, 3 sent, 4 exchange done,
5 δ2/b2 done, 6 g published.  Pass points: 8 top, 9 g ready, 10 x ready, 11 FMAs done,
12 acc published.  Printed as mean cycles between consecutive points over t in [8, 64).
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
buf = torch.zeros(4 * 64 * 16, dtype=torch.int64, device="cuda")
X, y = make_split(a.K * a.rows, "train", 0)
net = PNN(c.layers, c.act, c.init, a.K, c.lr)
net.set_kernel("resident")
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
L.pnn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
net.train_epoch(xd, yd)
torch.cuda.synchronize()
L.pnn_debug_set_trace(None)
tr = buf.cpu().numpy().reshape(4, 64, 16).astype(np.float64)
for cta in range(min(4, net.kernel_info()[0] and 4)):
    T = tr[cta, 8:64]
    if not T[:, 0].any():
        continue
    per = np.diff(T[:, 0]).mean()
    print(f"CTA {cta}: tail period {per:.0f} cyc/sample; pass period {np.diff(T[:, 8]).mean():.0f}")
    names = ["top", "acc_ready", "reduced", "sent", "exch_done", "d2_done", "g_pub"]
    seg = [T[:, i + 1] - T[:, i] for i in range(6)]
    print("  tail:", ", ".join(f"{names[i]}->{names[i+1]} {s.mean():.0f}" for i, s in enumerate(seg)))
    print("  tail g_pub->next top", np.mean(T[1:, 0] - T[:-1, 6]).round())
    pn = ["top", "g_ready", "x_ready", "fma_done", "acc_pub"]
    seg = [T[:, 8 + i + 1] - T[:, 8 + i] for i in range(4)]
    print("  pass:", ", ".join(f"{pn[i]}->{pn[i+1]} {s.mean():.0f}" for i, s in enumerate(seg)))
    print("  pass acc_pub(t) -> tail acc_ready(t):", np.mean(T[:, 1] - T[:, 12]).round(),
          " tail g_pub(t) -> pass g_ready(t+2):", np.mean(T[2:, 9] - T[:-2, 6]).round())
