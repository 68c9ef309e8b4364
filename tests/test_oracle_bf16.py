"""Pins of the oracle's bf16 mini-batch variant (a10; reading R25), CPU only.

* bf16 rounding: equals torch's float32 -> bfloat16 conversion (round to
  nearest even) on random values, exact ties and specials.
* one and two mini-batch steps on small ReLU/softmax and sigmoid/½-SSE nets:
  equal to an independent torch implementation of the same reading (torch's
  bf16 conversion at R25's rounding points, fp64 arithmetic) within fp32
  accumulation noise;
* η = 0 leaves the weights unchanged; the bf16 step stays within bf16 error of
  the fp32 mini-batch step (sanity of the rounding points).
"""
import numpy as np
import pytest
import torch

import oracle


def test_bf16_round_matches_torch():
    rng = np.random.default_rng(0)
    vals = np.concatenate([
        rng.normal(size=2000).astype(np.float32),
        (rng.normal(size=500) * 1e-30).astype(np.float32),
        (rng.normal(size=500) * 1e30).astype(np.float32),
        # exact ties: 1 + (2k+1)·2^-8 and their negatives
        np.array([1 + (2 * k + 1) * 2.0 ** -8 for k in range(64)], np.float32),
        -np.array([1 + (2 * k + 1) * 2.0 ** -8 for k in range(64)], np.float32),
        np.array([0.0, -0.0, np.inf, -np.inf, 3.0e38, 1e-45], np.float32),
    ])
    ref = torch.from_numpy(vals).to(torch.bfloat16).float().numpy()
    got = np.array([oracle.bf16_round(float(v)) for v in vals], np.float32)
    np.testing.assert_array_equal(got, ref)


def _bf(a):
    return torch.as_tensor(a, dtype=torch.float32).to(torch.bfloat16).to(torch.float64)


def _torch_bf16_steps(layers, act, params, X, y, lr, batch, epochs=1):
    """Independent reading-R25 reference in torch (fp64 arithmetic on bf16-rounded
    operands): forward/backward with weights fixed over each mini-batch."""
    P = torch.tensor(params, dtype=torch.float64)
    L = len(layers) - 1
    offs, o = [], 0
    for l in range(1, L + 1):
        offs.append(o)
        o += layers[l] * layers[l - 1] + layers[l]
    Xt = torch.tensor(X, dtype=torch.float64)
    for _ in range(epochs):
        for t0 in range(0, len(y), batch):
            xb = Xt[t0:t0 + batch]
            yb = y[t0:t0 + batch]
            B = xb.shape[0]
            Ws = [P[offs[l]:offs[l] + layers[l + 1] * layers[l]].view(layers[l + 1], layers[l]) for l in range(L)]
            bs = [P[offs[l] + layers[l + 1] * layers[l]:offs[l] + layers[l + 1] * layers[l] + layers[l + 1]]
                  for l in range(L)]
            Wb = [_bf(W.float()) for W in Ws]
            a = [_bf(xb.float())]                       # bf16 inputs of each layer
            xs = []
            for l in range(L):
                z = a[-1] @ Wb[l].T + bs[l]
                if act[l] == "softmax":
                    xl = torch.softmax(z, dim=1)
                elif act[l] == "relu":
                    xl = torch.relu(z)
                elif act[l] == "sigmoid":
                    xl = torch.sigmoid(z)
                else:
                    xl = torch.tanh(z)
                xs.append(xl)
                a.append(_bf(xl.float()))
            e = torch.zeros(B, layers[-1], dtype=torch.float64)
            e[torch.arange(B), torch.tensor(yb, dtype=torch.long)] = 1
            xo = xs[-1]
            if act[-1] == "softmax":
                d = xo - e
            else:
                d = (xo - e) * xo * (1 - xo)            # sigmoid output, ½-SSE (R11)
            grads = [None] * L
            for l in range(L - 1, -1, -1):
                db = _bf(d.float())
                grads[l] = (db.T @ a[l], d.sum(0))
                if l > 0:
                    h = xs[l - 1]
                    if act[l - 1] == "relu":
                        dphi = (h > 0).double()
                    elif act[l - 1] == "sigmoid":
                        dphi = h * (1 - h)
                    else:
                        dphi = 1 - h * h
                    d = (db @ Wb[l]) * dphi
            for l in range(L):
                gW, gb = grads[l]
                n = layers[l + 1] * layers[l]
                P[offs[l]:offs[l] + n] -= lr * (gW.reshape(-1) / B)
                P[offs[l] + n:offs[l] + n + layers[l + 1]] -= lr * (gb / B)
    return P.numpy()


@pytest.mark.parametrize("layers,act,batch,n", [
    ([12, 7, 5, 3], ["relu", "relu", "softmax"], 4, 10),
    ([9, 6, 4], ["sigmoid", "sigmoid"], 3, 7),
    ([16, 8, 4], ["tanh", "softmax"], 5, 12),
])
def test_bf16_minibatch_matches_torch_reference(layers, act, batch, n):
    rng = np.random.default_rng(1)
    p0 = oracle.init_params(layers, "he", 3)
    X = rng.random((n, layers[0])).astype(np.float32)
    y = rng.integers(0, layers[-1], n).astype(np.int32)
    got = oracle.train(layers, act, p0, X, y, 0.05, epochs=2, batch=batch, precision="bf16")
    ref = _torch_bf16_steps(layers, act, p0, X, y, 0.05, batch, epochs=2)
    np.testing.assert_allclose(got, ref, rtol=2e-5, atol=2e-6)


def test_bf16_eta_zero_and_close_to_fp32():
    layers, act = [20, 16, 10], ["relu", "softmax"]
    rng = np.random.default_rng(2)
    p0 = oracle.init_params(layers, "he", 5)
    X = rng.random((40, 20)).astype(np.float32)
    y = rng.integers(0, 10, 40).astype(np.int32)
    same = oracle.train(layers, act, p0, X, y, 0.0, batch=8, precision="bf16")
    np.testing.assert_array_equal(same, p0)
    b16 = oracle.train(layers, act, p0, X, y, 0.1, batch=8, precision="bf16")
    f32 = oracle.train(layers, act, p0, X, y, 0.1, batch=8)
    step = np.linalg.norm(f32 - p0)
    assert np.linalg.norm(b16 - f32) < 0.05 * step       # bf16 error ≪ the step itself
    assert np.linalg.norm(b16 - p0) > 0.5 * step
