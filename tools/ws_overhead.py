"""Fixed per-CTA overhead of the v12 SGD launch: time one wave (148 CNs) at several slice
lengths T; launch(T) = a + b·T, a = prologue/epilogue + pipeline fill/drain per wave."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_2304_09590_b200 import PNN
from workloads import CONFIGS
c = CONFIGS["C4"]
K = 148
res = []
for T in (16, 64, 256, 1024, 2048):
    n = K * T
    g = torch.Generator().manual_seed(0)
    X = torch.rand(n, 784, generator=g).cuda()
    y = torch.randint(0, 10, (n,), generator=g).int().cuda()
    net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
    net.set_variant("ws")
    for _ in range(2):
        net.train_epoch(X, y)
    torch.cuda.synchronize()
    net.kernel_timing(True)
    for _ in range(5):
        net.train_epoch(X, y)
    torch.cuda.synchronize()
    ms, L = net.kernel_timing(False)
    res.append((T, ms / L))
    print(f"T={T:5d}  SGD launch {ms / L:.4f} ms  per sample {ms / L / T * 1e3:.3f} us", flush=True)
    net.close()
T = np.array([r[0] for r in res], float); t = np.array([r[1] for r in res])
b, a = np.polyfit(T[-3:], t[-3:], 1)
print(f"fit (T >= 256): launch = {a*1e3:.1f} us + {b*1e6:.1f} ns x T  ({b*1e-3*1.965e9*1e3:.0f} cycles/sample at 1965 MHz)")
