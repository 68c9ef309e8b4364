"""§8(f) experiment harness on the GPU path (f1-f4), synthetic MNIST-shaped data.

    python tools/experiments.py curves [--config F1] [--K 1,2,10,20,30] [--epochs 20] [--lr 0.1]
        f1 + f2: per-epoch merged snapshot (children keep training unmerged,
        SPEC.md:378/413) -> accuracy / confidence / cost of the
        merged net and the mean over CNs (Fig.3/Fig.4/Fig.6 analogues).
    python tools/experiments.py sweep [--epochs 20]
        f3: activation sweep {tanh, leaky_relu, relu, sigmoid} x {SNN, 10-CN PNN},
        784-256-10, batch 50, η 0.05 (Fig.2).
    python tools/experiments.py table2 [--config C4] [--K 64] [--slots 1,2,4,8,16,32,64]
        f4: training time vs concurrently trained CN slots at fixed K (Table 2 analogue,
        PAPER.md:449-465), relative to 1 slot.

One JSON object per line on stdout.  Device-timed with CUDA events.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from datagen import make_split  # noqa: E402
from workloads import CONFIGS  # noqa: E402
from paper_2304_09590_b200 import PNN, PNN_BF16  # noqa: E402


def _net(cfg, K, act=None, lr=None, batch=None):
    net = PNN(cfg.layers, act or cfg.act, cfg.init, K, lr or cfg.lr, seed=0)
    b = cfg.batch if batch is None else batch
    if b > 1:
        net.set_minibatch(b, PNN_BF16 if cfg.precision == "bf16" else 0)
    return net


def _timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


DATA = "hard"


def run_curves(cfg, K, epochs, data, act=None, lr=None, tag="curves"):
    xd, yd, xt, yt = data
    net = _net(cfg, K, act, lr)
    for e in range(1, epochs + 1):
        ms = _timed(lambda: net.train_epoch(xd, yd))
        net.merge()
        acc, conf, cost = net.evaluate(xt, yt)
        cn = np.array([net.evaluate(xt, yt, subnet=i) for i in range(K)])
        print(json.dumps({"exp": tag, "config": cfg.name, "data": DATA, "act": act or list(cfg.act), "K": K,
                          "lr": lr or cfg.lr, "batch": cfg.batch, "epoch": e, "train_ms": ms,
                          "pnn": {"accuracy": acc, "confidence": conf, "cost": cost},
                          "cn_mean": {"accuracy": float(cn[:, 0].mean()), "confidence": float(cn[:, 1].mean()),
                                      "cost": float(cn[:, 2].mean())},
                          "cn_best_accuracy": float(cn[:, 0].max())}), flush=True)
    net.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["curves", "sweep", "table2"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--K", default=None)
    ap.add_argument("--epochs", type=int, default=None)
    ap.add_argument("--lr", type=float, default=None)
    ap.add_argument("--slots", default="1,2,4,8,16,32,64")
    ap.add_argument("--rows", type=int, default=None, help="override the training rows")
    ap.add_argument("--data", default="hard", choices=["hard", "easy"],
                    help="hard: the blended/noisier datagen variant (the default recipe is ~100%% separable)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    global DATA
    DATA = args.data

    if args.what in ("curves", "sweep"):
        cfg = CONFIGS[args.config or "F1"]
        n = args.rows or cfg.n_train
        X, y = make_split(n, "train", 0, hard=args.data == "hard")
        Xt, yt = make_split(cfg.n_test, "test", 0, hard=args.data == "hard")
        data = (torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(),
                torch.from_numpy(Xt).cuda(), torch.from_numpy(yt).cuda())
        epochs = args.epochs or cfg.epochs
        if args.what == "curves":
            for K in [int(k) for k in (args.K or "1,2,10,20,30").split(",")]:
                run_curves(cfg, K, epochs, data, lr=args.lr)
        else:
            for act in ("tanh", "leaky_relu", "relu", "sigmoid"):
                for K in [int(k) for k in (args.K or "1,10").split(",")]:
                    run_curves(cfg, K, epochs, data, act=[act, "softmax"], lr=args.lr or 0.05, tag="sweep")
    else:
        cfg = CONFIGS[args.config or "C4"]
        K = int(args.K or 64)
        S = cfg.n_train // cfg.K                        # the config's slice length
        X, y = make_split(K * S, "train", 0)
        xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
        base = None
        for slots in [int(s) for s in args.slots.split(",")]:
            net = _net(cfg, K)
            net.set_slots(slots)
            net.train_epoch(xd, yd)                     # warm-up
            ms = min(_timed(lambda: net.train_epoch(xd, yd)) for _ in range(3))
            base = base or ms
            print(json.dumps({"exp": "table2", "config": cfg.name, "K": K, "rows_per_cn": S, "slots": slots,
                              "epoch_ms": ms, "relative_time_pct": 100.0 * ms / base,
                              "samples_per_s": K * S / (ms / 1e3)}), flush=True)
            net.close()


if __name__ == "__main__":
    main()
