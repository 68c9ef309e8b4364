"""fp32 conditioning envelope — test infrastructure for the parity tolerance.

Per-sample SGD is an iteration: after thousands of sequential updates, two
correct fp32 implementations that merely sum in different orders drift apart,
and on ill-conditioned workloads (C2: N(0,1) init saturates the sigmoids, so
φ' = x(1-x) is quantised by fp32 rounding) they drift by more than the
north_star's 1e-4.  This module trains one CN with torch CPU fp32 (BLAS
summation order, the paper's per-sample SGD written with torch ops) so a test
can measure that spread: |torch_fp32 - oracle_fp32| is the disagreement of
two valid fp32 orderings.  A second measure needs no second implementation:
re-run the fp32 oracle from the same init perturbed by 1 ulp per parameter
(random direction) — how far the oracle itself moves is the precision to
which fp32 arithmetic determines the result at all (perturbation_envelope).
DESIGN.md §3 (R22) states the rule that uses them (tests/cnrule.py): a CN on a
smooth net passes if max-abs(GPU - oracle_fp32) <= max(1e-4, envelope), envelope =
the largest of the torch ordering and 64 1-ulp perturbation runs — the GPU,
another valid fp32 ordering, may differ from the oracle by no more than the oracle
differs from itself when fp32 does not determine the trajectory.
"""
import numpy as np
import torch


def torch_sgd_fp32(layers, act, params, X, y, lr, epochs=1, batch=1):
    """The paper's SGD (batch 1) or mini-batch GD (batch > 1: per-instance gradients summed
    by a BLAS matmul over the batch, averaged over its size, R14) in torch CPU fp32."""
    torch.set_num_threads(1)
    W, b, off = [], [], 0
    for l in range(1, len(layers)):
        nin, nout = layers[l - 1], layers[l]
        W.append(torch.tensor(params[off:off + nin * nout].reshape(nout, nin), dtype=torch.float32))
        off += nin * nout
        b.append(torch.tensor(params[off:off + nout], dtype=torch.float32))
        off += nout
    Xt = torch.tensor(np.asarray(X), dtype=torch.float32)
    eye = torch.eye(layers[-1], dtype=torch.float32)
    f = {"sigmoid": torch.sigmoid, "tanh": torch.tanh, "relu": torch.relu}
    L = len(layers) - 1
    for _ in range(epochs):
        for t0 in range(0, len(y), batch):
            xs = [Xt[t0:t0 + batch]]                     # rows = instances of the batch
            for l in range(L):
                z = xs[-1] @ W[l].T + b[l]
                xs.append(torch.softmax(z, 1) if act[l] == "softmax" else f[act[l]](z))
            o = xs[-1]
            e = eye[torch.as_tensor(np.asarray(y[t0:t0 + batch], np.int64))]
            if act[-1] == "softmax":
                d = o - e
            elif act[-1] == "sigmoid":
                d = (o - e) * o * (1 - o)
            elif act[-1] == "tanh":
                d = (o - e) * (1 - o * o)
            else:
                d = (o - e) * (o > 0).float()
            ds = [d]
            for l in range(L - 1, 0, -1):
                a = xs[l]
                g = {"sigmoid": a * (1 - a), "tanh": 1 - a * a, "relu": (a > 0).float()}[act[l - 1]]
                ds.insert(0, (ds[0] @ W[l]) * g)
            bsz = xs[0].shape[0]
            for l in range(L):
                if bsz == 1:
                    gl = lr * ds[l][0]
                    W[l] -= torch.outer(gl, xs[l][0])
                    b[l] -= gl
                else:
                    W[l] -= lr * ((ds[l].T @ xs[l]) / bsz)
                    b[l] -= lr * (ds[l].sum(0) / bsz)
    return np.concatenate([np.concatenate([W[l].ravel().numpy(), b[l].numpy()]) for l in range(L)])


def perturbation_envelope(orc, layers, act, params, X, y, lr, epochs=1, trials=64, seed=1, batch=1, threads=None):
    """max over `trials` of max-abs(oracle(params ± 1 ulp) - oracle(params)), fp32.

    With T exchangeable draws, a further draw exceeds their maximum with probability
    1/(T+1): at T = 64 a GPU result (another valid fp32 trajectory) outside the envelope
    is a ~1.5 % event, not a tolerance factor picked by hand.  Trials run in parallel
    (the oracle's C calls release the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    rng = np.random.default_rng(seed)
    p0 = np.asarray(params, np.float32)
    ref = orc.train(layers, act, p0, X, y, lr, epochs, batch=batch)
    dirs = [np.where(rng.random(p0.size) < 0.5, np.inf, -np.inf).astype(np.float32) for _ in range(trials)]

    def one(direction):
        pp = np.nextafter(p0, direction).astype(np.float32)
        return float(np.abs(orc.train(layers, act, pp, X, y, lr, epochs, batch=batch) - ref).max())

    n = threads or max(1, len(os.sched_getaffinity(0)))
    with ThreadPoolExecutor(max_workers=n) as ex:
        return max(ex.map(one, dirs))
