"""Per-CTA timeline of the tcgen05 GEMM (k_tcgemm.cuh debug trace; tools only):
standalone C5 step shapes through the debug hook, then the last step of a small C5 epoch."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2304_09590_b200 import load, PNN, PNN_BF16
from datagen import make_rows
from workloads import CONFIGS

L = load()
L.pnn_debug_tc_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5
L.pnn_debug_set_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(7 * 16384, dtype=torch.int64, device="cuda")
L.pnn_debug_set_trace(buf.data_ptr())
GHZ = 1.965


def report(name, t, nk):
    t = t[:24 * (len(t) // 24)].reshape(-1, 24)
    t = t[t[:, 1] != 0]
    if len(t) == 0:
        print(name, "no entries"); return
    c = t[:, 1:].astype(np.float64)
    d = lambda a, b: np.median(c[:, b - 1] - c[:, a - 1])
    kts = min(nk, 16)
    sp = [np.median(c[:, 4 + k] - c[:, 3 + k]) for k in range(kts - 1)] if kts > 1 else []
    skew = (t[:, 0].max() - t[:, 0].min()) / 1e3
    print(f"{name}: {len(t)} CTAs, launch skew {skew:.2f} us | prologue {d(1, 2):.0f} | griddep {d(2, 3):.0f} | "
          f"first stage {d(3, 4):.0f} | stage spacing med {np.median(sp) if sp else 0:.0f} (first 3: "
          f"{[int(x) for x in sp[:3]]}) | last stage->acc {np.median(c[:, 19] - c[:, 3 + kts - 1 + 1 - 1]):.0f} | "
          f"epilogue {d(20, 21):.0f} (tmem ld {d(20, 23):.0f}, chunks {d(23, 22):.0f}, tail {d(22, 21):.0f}) | total {d(1, 21):.0f} cycles = {d(1, 21) / GHZ / 1e3:.2f} us")


for name, Z, M, N, K, bn in [("F-shape K=784", 8, 1024, 64, 784, 64), ("F-shape K=1024", 8, 1024, 64, 1024, 64),
                             ("B5-shape", 8, 1024, 784, 64, 256)]:
    A = torch.randn(Z, M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(Z, N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(Z, M, N, device="cuda")
    for _ in range(3):
        buf.zero_()
        assert L.pnn_debug_tc_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), Z, M, N, K, bn) == 0
    report("standalone " + name, buf[:16384].cpu().numpy(), (K + 63) // 64)

c = CONFIGS["C5"]
R = 4
X, y = make_rows(0, 8 * 64 * R, "train", 0)
net = PNN(c.layers, c.act, c.init, 8, c.lr, seed=0)
net.set_minibatch(64, PNN_BF16)
xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
for _ in range(3):
    buf.zero_()
    net.train_epoch(xd, yd)
torch.cuda.synchronize()
h = buf.cpu().numpy()
for role, (nm, nk) in enumerate([("F1", 13), ("F2", 16), ("B4", 16), ("B3", 1), ("B5", 1)]):
    report("in-step " + nm, h[(role + 1) * 16384:(role + 2) * 16384], nk)
# the step's kernels on one clock: entry times (globaltimer) relative to F1's earliest CTA
g0 = h[16384:16384 + 24 * 64].reshape(-1, 24)[:, 0]
base = g0[g0 > 0].min()
for role, nm in enumerate(["F1", "F2", "B4", "B3", "B5"]):
    e = h[(role + 1) * 16384:(role + 1) * 16384 + 24 * 682].reshape(-1, 24)
    e = e[e[:, 1] != 0]
    ends = e[:, 0] + (e[:, 21] - e[:, 1]) / GHZ
    print(f"  {nm}: first entry {(e[:, 0].min() - base) / 1e3:7.2f} us, last entry {(e[:, 0].max() - base) / 1e3:7.2f}, "
          f"last end ~{(ends.max() - base) / 1e3:7.2f} us")
o = h[6 * 16384:6 * 16384 + 24 * 128].reshape(-1, 24)
o = o[o[:, 1] != 0]
c = o[:, 1:5].astype(np.float64)
cc = o.astype(np.float64)
print(f"  out_bwd detail: griddep->preloads issued {np.median(cc[:, 5] - cc[:, 2]):.0f} | ->z3 sums {np.median(cc[:, 6] - cc[:, 5]):.0f} | "
      f"->softmax/d3 {np.median(cc[:, 7] - cc[:, 6]):.0f} | ->barrier {np.median(cc[:, 3] - cc[:, 7]):.0f}")
print(f"in-step out_bwd: {len(o)} CTAs, entry {(o[:, 0].min() - base) / 1e3:.2f}..{(o[:, 0].max() - base) / 1e3:.2f} us | "
      f"griddep {np.median(c[:, 1] - c[:, 0]):.0f} | to delta3 {np.median(c[:, 2] - c[:, 1]):.0f} | "
      f"rest {np.median(c[:, 3] - c[:, 2]):.0f} cycles; last end ~"
      f"{(np.max(o[:, 0] + (c[:, 3] - c[:, 0]) / GHZ) - base) / 1e3:.2f} us")
L.pnn_debug_set_trace(None)
