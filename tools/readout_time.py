"""Merge and readout (predict of the C4 test set) times, CUDA events over 20 launches."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2304_09590_b200 import PNN
from workloads import CONFIGS
from datagen import make_split
c = CONFIGS["C4"]
K = 1024
net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
X, y = make_split(K * 8, "train", 0)
net.train_epoch(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
Xt, yt = make_split(10000, "test", 0)
xtd = torch.from_numpy(Xt).cuda()
ytd = torch.from_numpy(yt).cuda()
lab = torch.empty(10000, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
def t(name, fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s); e1.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us", flush=True)
t("merge", lambda: net.merge(s))
t("predict 10000", lambda: net.predict(xtd, lab, stream=s))
t("evaluate 10000", lambda: net.evaluate(xtd, ytd))
