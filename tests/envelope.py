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
DESIGN.md §3 (R22) states the rule that uses them: a CN passes if
max-abs(GPU - oracle_fp32) <= max(1e-4, 2 * envelope), envelope = the
largest of the torch ordering and three 1-ulp perturbation runs.
"""
import numpy as np
import torch


def torch_sgd_fp32(layers, act, params, X, y, lr, epochs=1):
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
        for t in range(len(y)):
            xs = [Xt[t]]
            for l in range(L):
                z = W[l] @ xs[-1] + b[l]
                xs.append(torch.softmax(z, 0) if act[l] == "softmax" else f[act[l]](z))
            o, e = xs[-1], eye[int(y[t])]
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
                ds.insert(0, (W[l].T @ ds[0]) * g)
            for l in range(L):
                gl = lr * ds[l]
                W[l] -= torch.outer(gl, xs[l])
                b[l] -= gl
    return np.concatenate([np.concatenate([W[l].ravel().numpy(), b[l].numpy()]) for l in range(L)])


def perturbation_envelope(orc, layers, act, params, X, y, lr, epochs=1, trials=3, seed=1, batch=1):
    """max over `trials` of max-abs(oracle(params ± 1 ulp) - oracle(params)), fp32."""
    rng = np.random.default_rng(seed)
    p0 = np.asarray(params, np.float32)
    ref = orc.train(layers, act, p0, X, y, lr, epochs, batch=batch)
    worst = 0.0
    for _ in range(trials):
        direction = np.where(rng.random(p0.size) < 0.5, np.inf, -np.inf).astype(np.float32)
        pp = np.nextafter(p0, direction).astype(np.float32)
        worst = max(worst, float(np.abs(orc.train(layers, act, pp, X, y, lr, epochs, batch=batch) - ref).max()))
    return worst


def check_minibatch_cns(orc, layers, act, init, K, lr, X, y, kids, okids, epochs, batch, tol=1e-4):
    """R22's per-CN rule for mini-batch runs: max-abs < tol, or <= 2x the oracle's own
    1-ulp perturbation envelope on that CN's slice (N(0,1)-init ReLU nets are as
    ill-conditioned in fp32 as C2)."""
    p0 = orc.init_params(layers, init, 0)
    start, count = orc.shard_bounds(len(y), K)
    report = []
    for i in range(K):
        err = float(np.abs(kids[i] - okids[i]).max())
        env = None
        if err >= tol:
            a, b = int(start[i]), int(start[i] + count[i])
            env = perturbation_envelope(orc, layers, act, p0, X[a:b], y[a:b], lr, epochs, batch=batch)
        report.append((i, err, env))
        assert err < tol or err <= 2 * env, f"CN {i}: max-abs {err:.3g}, fp32 envelope {env}"
    print("per-CN (index, max-abs vs oracle, fp32 envelope):", report)
    return report
