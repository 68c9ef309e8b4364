"""Where the C4 host-input step's time goes: train_epoch_host alone vs the full e2e step."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_2304_09590_b200 import PNN
from workloads import CONFIGS
from datagen import make_split
c = CONFIGS["C4"]
K, n = 1024, 1 << 20
g = torch.Generator().manual_seed(0)
xh = torch.rand(n, 784, generator=g).pin_memory()
yh = torch.randint(0, 10, (n,), generator=g).int().pin_memory()
net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
s = torch.cuda.current_stream()
for _ in range(2):
    net.train_epoch_host(xh, yh, s)
torch.cuda.synchronize()
for rep in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    net.train_epoch_host(xh, yh, s)
    t1 = time.perf_counter()
    e1.record(s)
    e1.synchronize()
    t2 = time.perf_counter()
    print(f"train_epoch_host: events {e0.elapsed_time(e1):.2f} ms, host call {1e3*(t1-t0):.2f} ms, to done {1e3*(t2-t0):.2f} ms", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for rep in range(4):
    net.train_epoch_host(xh, yh, s)
e1.record(s); e1.synchronize()
print(f"4 back-to-back calls: {e0.elapsed_time(e1)/4:.2f} ms per call")
xth = torch.rand(10000, 784, generator=g).pin_memory()
xtd = torch.empty(10000, 784, device="cuda")
labels = torch.empty(10000, dtype=torch.int32, device="cuda")
lab_h = torch.empty(10000, dtype=torch.int32).pin_memory()
def part(name, fn, reps=4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s); e1.synchronize()
    print(f"{name}: {e0.elapsed_time(e1)/reps:.3f} ms", flush=True)
part("merge", lambda: net.merge(s))
part("xt copy", lambda: xtd.copy_(xth, non_blocking=True))
part("predict", lambda: net.predict(xtd, labels, stream=s))
part("labels d2h", lambda: lab_h.copy_(labels, non_blocking=True))
def step():
    net.train_epoch_host(xh, yh, s)
    net.merge(s)
    xtd.copy_(xth, non_blocking=True)
    net.predict(xtd, labels, stream=s)
    lab_h.copy_(labels, non_blocking=True)
part("full step", step)
def step2():
    net.train_epoch_host(xh, yh, s)
    net.merge(s)
    net.predict(xtd, labels, stream=s)
part("step w/o test copies", step2)
ns2 = torch.cuda.Stream()
def stepA():
    net.train_epoch_host(xh, yh, s)
    net.merge(s)
    with torch.cuda.stream(ns2):
        xtd.copy_(xth, non_blocking=True)
    s.wait_stream(ns2)
    net.predict(xtd, labels, stream=s)
    lab_h.copy_(labels, non_blocking=True)
part("A: xt copy on a side stream", stepA)
def stepD():
    net.train_epoch_host(xh, yh, s)
    net.merge(s)
    torch.cuda.synchronize()
    xtd.copy_(xth, non_blocking=True)
    net.predict(xtd, labels, stream=s)
    lab_h.copy_(labels, non_blocking=True)
part("D: sync before xt copy", stepD)
def stepE():
    net.train_epoch_host(xh, yh, s)
    net.merge(s)
    xtd.copy_(xth, non_blocking=True)
    net.predict(xtd, labels, stream=s)
    lab_h.copy_(labels, non_blocking=True)
    torch.cuda.synchronize()
part("E: sync at step end", stepE)
