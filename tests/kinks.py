"""R24 kink accounting — test infrastructure for the ReLU parity rule.

SURVEY.md §8(c) R24 / DESIGN.md §3: on ReLU (and leaky-ReLU) nets, tiny GPU/oracle
rounding differences can flip the sign of a pre-activation z ≈ 0, switching φ'
between 1 and 0 (Eq.4's branch point, R9) for one unit of one sample;
that moves that CN's weights by up to ~η·|δ|·|x| ≈ 1e-3.  The rule: a per-CN
violation of the 1e-4 gate on such a net is accepted only if it coincides with a
LOGGED kink — a unit whose |z| < 1e-5 with a sign disagreement between the two
sides at the first divergent sample; otherwise it is a bug.

find_kink replays one CN through the C ABI (a K = 1 handle forced to the same kernel
variant, restarted from the same initial parameters, trained on prefixes of the CN's
sample sequence) and through the oracle, bisects for the first sample after which the
two disagree by more than `jump`, and reports the units of every ReLU-family layer
whose pre-activation at that sample is within `zeps` of 0 on either side, with both
sides' values (forward from each side's own parameters before that sample, fp64).
"""
from __future__ import annotations

import numpy as np
import torch

RELU_FAMILY = ("relu", "leaky_relu")


def _steps_per_epoch(m, batch):
    return (m + batch - 1) // batch


def _prefix_rows(Xi, yi, epochs, n, batch=1):
    """The first n update steps (single samples, or mini-batches of `batch` with the short
    last batch of each epoch, R14) of `epochs` passes over the slice, as a list of
    per-call (X, y) row ranges (each call is one pass from the slice start)."""
    m = len(yi)
    spe = _steps_per_epoch(m, batch)
    full, part = divmod(n, spe)
    calls = [(Xi, yi)] * min(full, epochs)
    if full < epochs and part:
        calls.append((Xi[:part * batch], yi[:part * batch]))
    return calls


def gpu_prefix(layers, act, lr, p0, Xi, yi, epochs, n, variant=None, kernel="auto", batch=1):
    from paper_2304_09590_b200 import PNN
    net = PNN(layers, act, "he", 1, lr, seed=0)
    net.set_kernel(kernel)
    if batch > 1:
        net.set_minibatch(batch)
    if variant is not None:
        net.set_variant(variant)
    net.set_params(p0)
    for X, y in _prefix_rows(Xi, yi, epochs, n, batch):
        net.train_epoch(torch.from_numpy(np.ascontiguousarray(X)).cuda(),
                        torch.from_numpy(np.ascontiguousarray(y)).cuda())
    torch.cuda.synchronize()
    out = net.get_params(0)
    net.close()
    return out


def oracle_prefix(orc, layers, act, lr, p0, Xi, yi, epochs, n, batch=1):
    p = np.asarray(p0, np.float32)
    for X, y in _prefix_rows(Xi, yi, epochs, n, batch):
        p = orc.train(layers, act, p, X, y, lr, 1, batch=batch)
    return p


def _epoch_checkpoints(orc, layers, act, lr, p0, Xi, yi, epochs, variant, kernel, batch):
    """Both sides' parameters after each epoch (index 0 = p0), one handle / one oracle run."""
    from paper_2304_09590_b200 import PNN
    net = PNN(layers, act, "he", 1, lr, seed=0)
    net.set_kernel(kernel)
    if batch > 1:
        net.set_minibatch(batch)
    if variant is not None:
        net.set_variant(variant)
    net.set_params(p0)
    xd = torch.from_numpy(np.ascontiguousarray(Xi)).cuda()
    yd = torch.from_numpy(np.ascontiguousarray(yi)).cuda()
    g, o = [np.asarray(p0, np.float32)], [np.asarray(p0, np.float32)]
    for _ in range(epochs):
        net.train_epoch(xd, yd)
        torch.cuda.synchronize()
        g.append(net.get_params(0))
        o.append(orc.train(layers, act, o[-1], Xi, yi, lr, 1, batch=batch))
    net.close()
    return g, o


def find_kink(orc, layers, act, lr, p0, Xi, yi, epochs=1, variant=None, kernel="auto", jump=1e-5, zeps=1e-5,
              batch=1):
    """Returns a dict: the first divergent update step (in the epochs × slice sequence;
    a sample, or a mini-batch), the errors just before / after it, and the near-zero units
    of the samples of that step: [(layer, unit, z_gpu, z_oracle, sign_disagrees)].
    Multi-epoch runs first find the first divergent epoch from per-epoch checkpoints of both
    sides, then bisect inside it from those checkpoints."""
    m = len(yi)
    spe = _steps_per_epoch(m, batch)
    e0 = 0
    pg0 = po0 = np.asarray(p0, np.float32)
    if epochs > 1:
        g, o = _epoch_checkpoints(orc, layers, act, lr, p0, Xi, yi, epochs, variant, kernel, batch)
        errs = [float(np.abs(a - b).max()) for a, b in zip(g, o)]
        if errs[-1] <= jump:
            return {"first_divergent": None, "err_total": errs[-1], "events": []}
        e0 = next(e for e in range(1, epochs + 1) if errs[e] > jump) - 1   # diverges during epoch e0
        pg0, po0 = g[e0], o[e0]

    def err(n):
        gp = gpu_prefix(layers, act, lr, pg0, Xi, yi, 1, n, variant, kernel, batch)
        op = oracle_prefix(orc, layers, act, lr, po0, Xi, yi, 1, n, batch)
        return float(np.abs(gp - op).max())

    if epochs == 1:
        e_total = err(spe)
        if e_total <= jump:
            return {"first_divergent": None, "err_total": e_total, "events": []}
    else:
        e_total = errs[-1]
    lo, hi = 0, spe                            # err(lo) <= jump < err(hi) (within epoch e0)
    if err(0) > jump:                          # already apart at the epoch start (tiny drift)
        lo = 0
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if err(mid) > jump:
            hi = mid
        else:
            lo = mid
    s = hi - 1                                 # the step of epoch e0 whose update diverged
    pg = gpu_prefix(layers, act, lr, pg0, Xi, yi, 1, s, variant, kernel, batch)
    po = oracle_prefix(orc, layers, act, lr, po0, Xi, yi, 1, s, batch)
    first = s * batch
    events = []
    for r in range(first, min(first + batch, m)):
        x = Xi[r].astype(np.float64)
        zg, _ = orc.forward(layers, act, pg.astype(np.float64), x)
        zo, _ = orc.forward(layers, act, po.astype(np.float64), x)
        for l, a in enumerate(act[:-1]):
            if a not in RELU_FAMILY:
                continue
            near = np.where((np.abs(zg[l]) < zeps) | (np.abs(zo[l]) < zeps))[0]
            for j in near:
                events.append((l + 1, int(j), float(zg[l][j]), float(zo[l][j]),
                               bool(np.sign(zg[l][j]) != np.sign(zo[l][j]))))
    return {"first_divergent": int(e0 * spe + s), "epoch": int(e0), "row": int(first), "err_before": err(s),
            "err_after": err(s + 1), "err_total": e_total, "events": events}


def has_kink(report) -> bool:
    """R24: the violation coincides with a logged kink — a near-zero unit at the first
    divergent sample (a sign disagreement there, or |z| < zeps on both sides: the
    fp32 forward inside the kernel rounds differently from this fp64 replay)."""
    return report["first_divergent"] is not None and len(report["events"]) > 0
