"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names the passage it pins and the kind of pin: a hand-computed
closed form, central finite differences, a library routine (torch fp64
autograd + torch.optim.SGD), or an invariant of the method.
"""
import math

import numpy as np
import pytest
import torch

from datagen import make_split

ACT_PAIRS = [  # (hidden, output) — every activation/loss pair the configs use
    ("sigmoid", "sigmoid"),   # C1, C2: ½-SSE (R11)
    ("tanh", "softmax"),      # C3: softmax + CE (Eq.10)
    ("relu", "softmax"),      # C4, C5
    ("sigmoid", "softmax"),
    ("tanh", "tanh"),
    ("relu", "sigmoid"),
    ("leaky_relu", "softmax"),   # f3 (slope 0.01, R30)
]


def sig(z):
    return 1.0 / (1.0 + math.exp(-z))


# --------------------------------------------------------------------------
# Hand-computed closed forms (Eqs.2-13)
# --------------------------------------------------------------------------
def test_hand_111_sigmoid_mse(orc):
    """1-1-1 sigmoid/sigmoid net, ½-SSE (R11): every quantity written out by
    the scalar chain rule, then one SGD step (Eqs.12-13)."""
    x0, w1, b1, w2, b2, eta = 0.5, 0.4, 0.1, -0.3, 0.2, 0.7
    params = np.array([w1, b1, w2, b2])
    zs, xs = orc.forward([1, 1, 1], ["sigmoid", "sigmoid"], params, [x0])
    a1 = sig(0.3)                       # z1 = 0.4*0.5 + 0.1
    a2 = sig(-0.3 * a1 + 0.2)
    assert zs[0][0] == pytest.approx(0.3, abs=1e-15)
    assert xs[0][0] == pytest.approx(a1, abs=1e-15)
    assert xs[1][0] == pytest.approx(a2, abs=1e-15)
    # label 0 ⇒ e = 1.  C = ½(a2-1)^2; δ2 = (a2-1)·a2(1-a2); δ1 = w2 δ2 · a1(1-a2)
    d2 = (a2 - 1.0) * a2 * (1.0 - a2)
    d1 = w2 * d2 * a1 * (1.0 - a1)
    assert orc.cost([1, 1, 1], ["sigmoid", "sigmoid"], params, [x0], 0) == pytest.approx(
        0.5 * (a2 - 1) ** 2, abs=1e-15)
    new = orc.train([1, 1, 1], ["sigmoid", "sigmoid"], params, np.array([[x0]]), np.array([0]),
                    eta, dtype=np.float64)
    exp = [w1 - eta * d1 * x0, b1 - eta * d1, w2 - eta * d2 * a1, b2 - eta * d2]
    np.testing.assert_allclose(new, exp, rtol=0, atol=1e-15)


def test_hand_222_softmax_full_jacobian(orc):
    """2-2-2 tanh/softmax net with CE.  δ^L is computed here through the FULL
    softmax Jacobian, ∂C/∂z_k = Σ_i (-e_i/x_i)·x_i(δ_ik - x_k), not through
    Eq.10's shortcut x - e — so this also pins Eq.10."""
    W1 = np.array([[0.3, -0.2], [0.5, 0.1]]); b1 = np.array([0.05, -0.1])
    W2 = np.array([[-0.4, 0.6], [0.2, 0.3]]); b2 = np.array([0.0, 0.15])
    x0 = np.array([0.8, -0.6]); label = 1; eta = 0.3
    params = np.concatenate([W1.ravel(), b1, W2.ravel(), b2])
    z1 = [W1[k, 0] * x0[0] + W1[k, 1] * x0[1] + b1[k] for k in range(2)]
    a1 = [math.tanh(z) for z in z1]
    z2 = [W2[k, 0] * a1[0] + W2[k, 1] * a1[1] + b2[k] for k in range(2)]
    ez = [math.exp(z) for z in z2]
    a2 = [e / sum(ez) for e in ez]
    e = [0.0, 1.0]
    d2 = [sum((-e[i] / a2[i]) * a2[i] * ((1.0 if i == k else 0.0) - a2[k]) for i in range(2))
          for k in range(2)]
    d1 = [(W2[0, j] * d2[0] + W2[1, j] * d2[1]) * (1 - a1[j] ** 2) for j in range(2)]
    zs, xs = orc.forward([2, 2, 2], ["tanh", "softmax"], params, x0)
    np.testing.assert_allclose(xs[1], a2, atol=1e-15)
    np.testing.assert_allclose(zs[1], z2, atol=1e-15)
    new = orc.train([2, 2, 2], ["tanh", "softmax"], params, x0[None], np.array([label]), eta,
                    dtype=np.float64)
    nW1 = W1 - eta * np.outer(d1, x0); nb1 = b1 - eta * np.array(d1)
    nW2 = W2 - eta * np.outer(d2, a1); nb2 = b2 - eta * np.array(d2)
    np.testing.assert_allclose(new, np.concatenate([nW1.ravel(), nb1, nW2.ravel(), nb2]),
                               atol=1e-14)


def test_relu_branch_points(orc):
    """Eq.4: φ(z)=z for z≥0, 0 for z<0; R9: ReLU'(0)=0 so a unit sitting at
    exactly z=0 passes no gradient (its incoming weights stay put)."""
    # 1-2-1 net: unit 0 sits at z=0 exactly, unit 1 at z=-1
    params = np.array([0.0, 1.0, 0.0, -2.0,      # W1 (2x1), b1
                       1.0, 1.0, 0.0])           # W2 (1x2), b2
    zs, xs = orc.forward([1, 2, 1], ["relu", "sigmoid"], params, [1.0])
    assert list(zs[0]) == [0.0, -1.0] and list(xs[0]) == [0.0, 0.0]
    new = orc.train([1, 2, 1], ["relu", "sigmoid"], params, np.array([[1.0]]), np.array([0]),
                    0.5, dtype=np.float64)
    np.testing.assert_array_equal(new[:4], params[:4])         # no gradient through z<=0
    params2 = np.array([3.0, -1.0, 0.0, 0.0, 1.0, 1.0, 0.0])
    zs, xs = orc.forward([1, 2, 1], ["relu", "sigmoid"], params2, [1.0])
    assert list(xs[0]) == [3.0, 0.0]


def test_leaky_relu_branch_points(orc):
    """Leaky ReLU (slope 0.01 by reading R30): φ(-1) = -0.01,
    φ(0) = 0; at z = 0 the left slope 0.01 applies (as R9 takes ReLU'(0) = 0), so
    unlike ReLU the unit at z = 0 passes 0.01 of its gradient (torch's
    LeakyReLU derivative at 0 is also the left one)."""
    params = np.array([0.0, 1.0, 0.0, -2.0, 1.0, 1.0, 0.0])
    zs, xs = orc.forward([1, 2, 1], ["leaky_relu", "sigmoid"], params, [1.0])
    assert list(zs[0]) == [0.0, -1.0]
    assert xs[0][0] == 0.0 and xs[0][1] == -0.01
    new = orc.train([1, 2, 1], ["leaky_relu", "sigmoid"], params, np.array([[1.0]]), np.array([0]),
                    0.5, dtype=np.float64)
    x2 = 1.0 / (1.0 + np.exp(-(0.0 * 1.0 + (-0.01) * 1.0)))
    d2 = (x2 - 1.0) * x2 * (1.0 - x2)                       # Eq.9 with ½-SSE (R11)
    np.testing.assert_allclose(new[0], 0.0 - 0.5 * (1.0 * d2 * 0.01) * 1.0, rtol=1e-12)
    np.testing.assert_allclose(new[1], 1.0 - 0.5 * (1.0 * d2 * 0.01) * 1.0, rtol=1e-12)
    t = torch.tensor([0.0, -1.0], dtype=torch.float64, requires_grad=True)
    torch.nn.functional.leaky_relu(t, 0.01).sum().backward()
    assert list(t.grad.numpy()) == [0.01, 0.01]


def test_softmax_closed_forms(orc):
    """Eq.5: zero-weight/zero-bias net → uniform 1/10; CE of the
    uniform output = ln 10 (Eq.6); [1000,1000] → [.5,.5] without overflow (R4);
    outputs sum to 1 and are shift-invariant."""
    P = orc.param_count([784, 16, 10])
    zs, xs = orc.forward([784, 16, 10], ["relu", "softmax"], np.zeros(P), np.random.rand(784))
    np.testing.assert_allclose(xs[1], 0.1, atol=1e-16)
    assert orc.cost([784, 16, 10], ["relu", "softmax"], np.zeros(P), np.random.rand(784), 3) == \
        pytest.approx(math.log(10), abs=1e-14)
    p = np.array([0.0, 0.0, 1000.0, 1000.0])        # 1-2 softmax layer: W=0, b=1000
    _, xs = orc.forward([1, 2], ["softmax"], p, [0.3])
    np.testing.assert_allclose(xs[0], [0.5, 0.5], atol=0)
    rng = np.random.default_rng(1)
    W = rng.normal(size=(10, 5)); b = rng.normal(size=10) * 3
    x = rng.normal(size=5)
    _, xs1 = orc.forward([5, 10], ["softmax"], np.concatenate([W.ravel(), b]), x)
    _, xs2 = orc.forward([5, 10], ["softmax"], np.concatenate([W.ravel(), b + 123.0]), x)
    assert abs(xs1[0].sum() - 1) < 1e-12
    np.testing.assert_allclose(xs1[0], xs2[0], atol=1e-12)
    _, xs32 = orc.forward([5, 10], ["softmax"], np.concatenate([W.ravel(), b]), x, dtype=np.float32)
    assert abs(float(xs32[0].sum()) - 1) < 1e-6


# --------------------------------------------------------------------------
# Finite differences (Eqs.7-11): the update with η=1 recovers -∂C/∂θ
# --------------------------------------------------------------------------
@pytest.mark.parametrize("hid,out", ACT_PAIRS)
@pytest.mark.parametrize("layers", [[4, 5, 3], [4, 5, 4, 3]])
def test_gradient_matches_central_differences(orc, hid, out, layers):
    rng = np.random.default_rng(hash((hid, out, len(layers))) % 2**32)
    act = [hid] * (len(layers) - 2) + [out]
    P = orc.param_count(layers)
    params = rng.normal(scale=0.7, size=P)
    x0 = rng.uniform(0, 1, size=layers[0])
    label = int(rng.integers(0, layers[-1]))
    eta = 1.0
    after = orc.train(layers, act, params, x0[None], np.array([label]), eta, dtype=np.float64)
    grad = (params - after) / eta
    h = 1e-6
    fd = np.empty(P)
    for i in range(P):
        pp = params.copy(); pp[i] += h
        pm = params.copy(); pm[i] -= h
        fd[i] = (orc.cost(layers, act, pp, x0, label) - orc.cost(layers, act, pm, x0, label)) / (2 * h)
    np.testing.assert_allclose(grad, fd, rtol=1e-5, atol=1e-7)


# --------------------------------------------------------------------------
# Library pin: torch fp64 autograd + torch.optim.SGD, per-sample and mini-batch
# --------------------------------------------------------------------------
def _torch_net(layers, act, params):
    mods = []
    off = 0
    for l in range(1, len(layers)):
        lin = torch.nn.Linear(layers[l - 1], layers[l]).double()
        nw = layers[l - 1] * layers[l]
        with torch.no_grad():
            lin.weight.copy_(torch.from_numpy(params[off:off + nw].reshape(layers[l], layers[l - 1])))
            lin.bias.copy_(torch.from_numpy(params[off + nw:off + nw + layers[l]]))
        off += nw + layers[l]
        mods.append(lin)
        a = act[l - 1]
        if a == "sigmoid":
            mods.append(torch.nn.Sigmoid())
        elif a == "tanh":
            mods.append(torch.nn.Tanh())
        elif a == "relu":
            mods.append(torch.nn.ReLU())
        elif a == "leaky_relu":
            mods.append(torch.nn.LeakyReLU(0.01))
    return torch.nn.Sequential(*mods)


def _torch_flat(net):
    return np.concatenate([t.detach().numpy().ravel() for m in net
                           if isinstance(m, torch.nn.Linear) for t in (m.weight, m.bias)])


def _torch_loss(out, yb, softmax_out, n_out, reduction):
    if softmax_out:   # Eq.6 CE on softmax(z): torch's cross_entropy takes the logits
        return torch.nn.functional.cross_entropy(out, yb, reduction=reduction)
    e = torch.nn.functional.one_hot(yb, n_out).double()
    per = 0.5 * ((out - e) ** 2).sum(dim=1)
    return per.sum() if reduction == "sum" else per.mean()


@pytest.mark.parametrize("hid,out", ACT_PAIRS)
@pytest.mark.parametrize("layers", [[12, 7, 5], [12, 9, 6, 5]])
def test_sgd_shard_matches_torch_fp64(orc, hid, out, layers):
    """Sequential per-sample SGD over a 120-sample slice ==
    torch fp64 autograd + SGD(lr), to 1e-10."""
    rng = np.random.default_rng(7)
    act = [hid] * (len(layers) - 2) + [out]
    P = orc.param_count(layers)
    params = rng.normal(scale=0.5, size=P)
    X = rng.uniform(0, 1, size=(120, layers[0]))
    y = rng.integers(0, layers[-1], size=120).astype(np.int32)
    eta = 0.05
    ours = orc.train(layers, act, params, X, y, eta, epochs=2, dtype=np.float64)
    net = _torch_net(layers, act, params)
    opt = torch.optim.SGD(net.parameters(), lr=eta)
    Xt, yt = torch.from_numpy(X), torch.from_numpy(y).long()
    for _ in range(2):
        for t in range(len(y)):
            opt.zero_grad()
            _torch_loss(net(Xt[t:t + 1]), yt[t:t + 1], out == "softmax", layers[-1], "sum").backward()
            opt.step()
    np.testing.assert_allclose(ours, _torch_flat(net), rtol=0, atol=1e-10)


@pytest.mark.parametrize("hid,out", [("relu", "softmax"), ("sigmoid", "sigmoid")])
def test_minibatch_matches_torch_mean(orc, hid, out):
    """Mini-batch GD: gradients averaged over the batch before the update
    (PAPER.md:134); the short last batch (50 = 6·8 + 2) averages over 2 (R14)."""
    layers = [10, 8, 4]
    rng = np.random.default_rng(3)
    P = orc.param_count(layers)
    params = rng.normal(scale=0.5, size=P)
    X = rng.uniform(0, 1, size=(50, 10)); y = rng.integers(0, 4, size=50).astype(np.int32)
    ours = orc.train(layers, [hid, out], params, X, y, 0.1, batch=8, dtype=np.float64)
    net = _torch_net(layers, [hid, out], params)
    opt = torch.optim.SGD(net.parameters(), lr=0.1)
    Xt, yt = torch.from_numpy(X), torch.from_numpy(y).long()
    for t0 in range(0, 50, 8):
        opt.zero_grad()
        _torch_loss(net(Xt[t0:t0 + 8]), yt[t0:t0 + 8], out == "softmax", 4, "mean").backward()
        opt.step()
    np.testing.assert_allclose(ours, _torch_flat(net), rtol=0, atol=1e-12)


def test_update_edge_cases(orc):
    """Eqs.12-13: η=0 leaves the network unchanged; a small step descends."""
    layers = [6, 5, 3]
    rng = np.random.default_rng(11)
    params = rng.normal(size=orc.param_count(layers))
    x = rng.uniform(size=(1, 6)); y = np.array([2], np.int32)
    for act in (["sigmoid", "sigmoid"], ["tanh", "softmax"]):
        np.testing.assert_array_equal(orc.train(layers, act, params, x, y, 0.0, dtype=np.float64), params)
        new = orc.train(layers, act, params, x, y, 1e-3, dtype=np.float64)
        assert orc.cost(layers, act, new, x[0], 2) < orc.cost(layers, act, params, x[0], 2)


def test_fp32_oracle_inside_fp64_envelope(orc):
    """The fp32 build (the parity gate) stays within 1e-5 of the fp64 truth on
    the C1 workload — the drift envelope a correct GPU must also sit in."""
    X, y = make_split(1000, "train", 0)
    p0 = orc.init_params([784, 16, 10], "uniform", 0)
    w32 = orc.train([784, 16, 10], ["sigmoid", "sigmoid"], p0, X, y, 0.1, dtype=np.float32)
    w64 = orc.train([784, 16, 10], ["sigmoid", "sigmoid"], p0.astype(np.float64), X, y, 0.1,
                    dtype=np.float64)
    assert np.abs(w32 - w64).max() < 1e-5


# --------------------------------------------------------------------------
# Slicing, merge, readout invariants
# --------------------------------------------------------------------------
@pytest.mark.parametrize("N,K", [(1000, 1), (60000, 4), (60000, 32), (1 << 20, 1024), (103, 8), (7, 7)])
def test_shards_disjoint_and_cover(orc, N, K):
    start, count = orc.shard_bounds(N, K)
    assert start[0] == 0 and (start[1:] == start[:-1] + count[:-1]).all()
    assert count.sum() == N and count.max() - count.min() <= 1
    assert (np.diff(count) <= 0).all()          # longer slices first (R17)


def test_merge_invariants(orc):
    rng = np.random.default_rng(5)
    P = 1001
    W = rng.normal(size=P).astype(np.float32)
    for K in (1, 2, 4, 8, 32, 1024):            # clones → exact identity (R18)
        np.testing.assert_array_equal(orc.merge(np.tile(W, (K, 1))), W)
    np.testing.assert_array_equal(orc.merge(np.stack([W, -W])), np.zeros(P, np.float32))
    kids = rng.normal(size=(7, P)).astype(np.float32)
    m = orc.merge(kids)
    np.testing.assert_array_equal(m, orc.merge(kids[rng.permutation(7)]))
    np.testing.assert_array_equal(m, np.mean(kids.astype(np.float64), axis=0).astype(np.float32))


def test_pnn_k1_is_snn_and_duplicated_shards(orc):
    """K=1 PNN == SNN (the TrainableNetwork interchangeability);
    K clones on duplicated identical slices → the merge equals any child."""
    layers, act = [784, 16, 10], ["sigmoid", "sigmoid"]
    X, y = make_split(300, "train", 0)
    p0 = orc.init_params(layers, "uniform", 0)
    kids, merged = orc.train_pnn(layers, act, "uniform", 1, 0.1, 0, X, y)
    snn = orc.train(layers, act, p0, X, y, 0.1)
    np.testing.assert_array_equal(kids[0], snn)
    np.testing.assert_array_equal(merged, snn)
    Xd, yd = np.tile(X[:75], (4, 1)), np.tile(y[:75], 4)
    kids, merged = orc.train_pnn(layers, act, "uniform", 4, 0.1, 0, Xd, yd)
    for k in kids:
        np.testing.assert_array_equal(k, kids[0])
    np.testing.assert_array_equal(merged, kids[0])


def test_predict_ties_and_shift(orc):
    """Readout = argmax, ties → lowest index (R19); argmax is invariant under
    a constant shift of the logits."""
    layers = [784, 16, 10]
    P = orc.param_count(layers)
    X, _ = make_split(50, "test", 0)
    assert (orc.predict(layers, ["relu", "softmax"], np.zeros(P), X) == 0).all()
    p = np.zeros(P); p[-10:] = [0, 3, 0, 3, 0, 0, 0, 0, 0, 0]
    assert (orc.predict(layers, ["relu", "softmax"], p, X) == 1).all()
    rng = np.random.default_rng(2)
    p = rng.normal(size=P)
    l1 = orc.predict(layers, ["relu", "softmax"], p, X)
    p2 = p.copy(); p2[-10:] += 17.0
    np.testing.assert_array_equal(l1, orc.predict(layers, ["relu", "softmax"], p2, X))
    _, logits = orc.predict(layers, ["relu", "softmax"], p, X, return_logits=True)
    np.testing.assert_array_equal(l1, np.argmax(logits, axis=1))


# --------------------------------------------------------------------------
# Init (R15, R16)
# --------------------------------------------------------------------------
def test_init_determinism_and_moments(orc):
    layers = [784, 128, 10]
    a = orc.init_params(layers, "normal", 42)
    np.testing.assert_array_equal(a, orc.init_params(layers, "normal", 42))
    assert not np.array_equal(a, orc.init_params(layers, "normal", 43))
    assert abs(a.mean()) < 0.02 and abs(a.var() - 1) < 0.05          # N(0,1)
    u = orc.init_params(layers, "uniform", 1)
    assert u.min() >= -0.5 and u.max() < 0.5
    assert abs(u.mean()) < 0.01 and abs(u.var() - 1 / 12) < 0.003
    for init, var in (("xavier", 2 / (784 + 128)), ("he", 2 / 784)):
        p = orc.init_params(layers, init, 3)
        W1 = p[:784 * 128]
        assert abs(W1.var() / var - 1) < 0.03
        assert (p[784 * 128:784 * 128 + 128] == 0).all()              # biases 0 (R15)
    us = np.array([orc.uniform(9, 1, 0, i) for i in range(20000)])
    assert 0 <= us.min() and us.max() < 1 and abs(us.mean() - 0.5) < 0.01
    # Box–Muller: one value written out from its two uniforms
    u1, u2 = orc.uniform(9, 2, 1, 5, 0), orc.uniform(9, 2, 1, 5, 1)
    assert orc.normal(9, 2, 1, 5) == math.sqrt(-2 * math.log(1 - u1)) * math.cos(2 * math.pi * u2)


def test_fp32_ordering_envelope():
    """tests/envelope.py (torch CPU fp32, BLAS order) is itself pinned: on the
    well-conditioned C1 workload it agrees with the fp32 oracle to 2e-5; on C2
    slice 3 (N(0,1) init → saturated sigmoids) two valid fp32 orderings already
    disagree by more than 1e-4 — the reason for the envelope rule (R22)."""
    import oracle
    from datagen import make_rows
    from tests.envelope import torch_sgd_fp32
    from workloads import CONFIGS
    c = CONFIGS["C1"]
    X, y = make_split(1000, "train", 0)
    p0 = oracle.init_params(c.layers, c.init, 0)
    d = np.abs(torch_sgd_fp32(c.layers, c.act, p0, X, y, c.lr) - oracle.train(c.layers, c.act, p0, X, y, c.lr))
    assert d.max() < 2e-5
    c = CONFIGS["C2"]
    s, n = oracle.shard_bounds(c.n_train, c.K)
    X, y = make_rows(int(s[3]), int(n[3]))
    p0 = oracle.init_params(c.layers, c.init, 0)
    d = np.abs(torch_sgd_fp32(c.layers, c.act, p0, X, y, c.lr) - oracle.train(c.layers, c.act, p0, X, y, c.lr))
    assert d.max() > 1e-4
    # and the oracle itself moves by > 1e-4 under 1-ulp perturbations of the init (C2 slice 3),
    # but by < 1e-5 on C1
    from tests.envelope import perturbation_envelope
    assert perturbation_envelope(oracle, c.layers, c.act, p0, X, y, c.lr, trials=1) > 1e-4
    c1 = CONFIGS["C1"]
    X1, y1 = make_split(1000, "train", 0)
    assert perturbation_envelope(oracle, c1.layers, c1.act, oracle.init_params(c1.layers, c1.init, 0),
                                 X1, y1, c1.lr, trials=1) < 1e-5


def test_fp32_ordering_envelope_minibatch():
    """The mini-batch arm of tests/envelope.py (batch gradient as one BLAS matmul,
    averaged over the batch, R14 short last batch) agrees with the fp32 oracle's
    mini-batch GD to 1e-6 on a well-conditioned tanh net with a ragged last batch; a
    transposed or unscaled batch gradient would miss by orders of magnitude."""
    import oracle
    X, y = make_split(203, "train", 0)
    layers, act = [784, 32, 10], ["tanh", "softmax"]
    p0 = oracle.init_params(layers, "xavier", 0)
    from tests.envelope import torch_sgd_fp32
    d = np.abs(torch_sgd_fp32(layers, act, p0, X, y, 0.05, 2, batch=7)
               - oracle.train(layers, act, p0, X, y, 0.05, 2, batch=7))
    assert d.max() < 1e-6


def test_r34_rejects_an_inaccurate_result():
    """R34 (tests/cnrule.py) passes a CN beyond the fp32 envelope only if the GPU is no
    farther from the fp64 run of the same algorithm than the fp32 oracle is: a result off
    by 2e-3 in one weight is rejected, the fp32 oracle's own result is accepted."""
    import oracle
    from tests.cnrule import cn_bound
    X, y = make_split(120, "train", 0)
    layers, act = [784, 32, 10], ["sigmoid", "sigmoid"]
    p0 = oracle.init_params(layers, "uniform", 0)
    okid = oracle.train(layers, act, p0, X, y, 0.1)
    bad = okid.copy()
    bad[5] += 2e-3
    bound, info = cn_bound(oracle, None, layers, act, "uniform", 0.1, X, y, 2e-3, okid, 1, kid=bad)
    assert bound < 2e-3 and info["fp64"]["gpu_vs_fp64"] > info["fp64"]["oracle32_vs_fp64"]
    bound, info = cn_bound(oracle, None, layers, act, "uniform", 0.1, X, y, 2e-3, okid, 1, kid=okid)
    assert bound == 2e-3
