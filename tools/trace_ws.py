"""clock64 timeline of the warp-specialised variant (v12, k_ws.cu), CTA 0, from a
-DPNN_WS_TRACE build (PNN_LIB=...).  Chain warp 0 per sample c: 0 loop top, 1 after aready(c),
2 after the partial-logit barrier, 3 gready(c) arrived.  Sweep warp 0 per pair p: 4 step top,
5 F(2p, 2p+1) done, 6 U-pair after its gready wait, 7 U-pair done.

    PNN_LIB=.../libpnn_tr.so python tools/trace_ws.py --K 148 --rows 256
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
ap.add_argument("--K", type=int, default=148)
ap.add_argument("--rows", type=int, default=256)
a = ap.parse_args()
c = CONFIGS["C4"]
L = load()
L.pnn_debug_set_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(256 * 8, dtype=torch.int64, device="cuda")
X, y = make_split(a.K * a.rows, "train", 0)
net = PNN(c.layers, c.act, c.init, a.K, c.lr)
net.set_variant("ws")
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
net.train_epoch(xd, yd)
L.pnn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
net.train_epoch(xd, yd)
torch.cuda.synchronize()
L.pnn_debug_set_trace(None)
tr = buf.cpu().numpy().reshape(256, 8).astype(np.float64)
ch = tr[32:200]
print("chain per sample (cycles): period %.0f" % np.median(np.diff(ch[:, 0])))
print("  waits (top -> aready) %.0f | z1+logits+barrier %.0f | softmax+delta+g %.0f | tail->next top %.0f" % (
    np.median(ch[:, 1] - ch[:, 0]), np.median(ch[:, 2] - ch[:, 1]), np.median(ch[:, 3] - ch[:, 2]),
    np.median(ch[1:, 0] - ch[:-1, 3])))
sw = tr[16:100]
print("sweep warp 0 per pair: period %.0f" % np.median(np.diff(sw[:, 4])))
print("  F-pair %.0f | F end -> U wait done %.0f | U-pair %.0f" % (
    np.median(sw[:, 5] - sw[:, 4]), np.median(sw[:, 6] - sw[:, 5]), np.median(sw[:, 7] - sw[:, 6])))
