"""GPU parity of the resident fp32 mini-batch kernel (k_mbres.cu: one persistent launch
per epoch, W¹ in the registers of a cluster of ⌈H/32⌉ CTAs) against the fp32 oracle's
mini-batch GD (R14 short last batch averaged over its size).

Tolerance: max-abs 1e-4 on every parameter (BASELINE.json north_star), a CN over it
only with a recorded cause (tests/cnrule.py: a logged ReLU kink, R24, or the fp32
envelope of a smooth net, R22); the merged net within the mean of the per-CN bounds.
The kernel applies W¹'s batch gradient row by row (w += (−η δ1_b / bsz)·x_b) instead
of sum-then-scale, a rounding-order difference.
"""
import numpy as np
import pytest
import torch

from datagen import make_split
from workloads import CONFIGS

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def _run(orc, layers, act, init, K, lr, n, batch, epochs=1):
    from paper_2304_09590_b200 import PNN
    X, y = make_split(n, "train", 0)
    X = np.ascontiguousarray(X[:, :layers[0]])
    net = PNN(layers, act, init, K, lr, seed=0)
    net.set_minibatch(batch)
    assert tuple(net.kernel_info()) == (6, 1)
    xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    for _ in range(epochs):
        net.train_epoch(xd, yd)
    net.merge()
    torch.cuda.synchronize()
    kids = np.stack([net.get_params(i) for i in range(K)])
    okids, omerged = orc.train_pnn(layers, act, init, K, lr, 0, X, y, epochs=epochs, batch=batch, threads=8)
    from tests.cnrule import check_cns, check_merged
    bounds = check_cns(orc, net, layers, act, init, K, lr, X, y, kids, okids, epochs, batch)
    check_merged(net.get_params(-1), omerged, bounds)


def test_f1_shape_two_epochs(orc):
    c = CONFIGS["F1"]
    _run(orc, c.layers, c.act, c.init, 4, c.lr, 4 * 260 + 3, c.batch, epochs=2)


@pytest.mark.parametrize("layers,act,batch", [
    ([784, 100, 10], ["sigmoid", "sigmoid"], 16),       # 4 CTAs, the last one 4 units
    ([784, 38, 4], ["tanh", "softmax"], 2),             # 2 CTAs, 4 outputs, batch 2
    ([784, 256, 16], ["leaky_relu", "softmax"], 64),    # widest, 16 outputs, batch 64
    ([772, 32, 10], ["sigmoid", "softmax"], 7),         # 1 CTA, D < 784
])
def test_shapes(orc, layers, act, batch):
    _run(orc, layers, act, "xavier", 3, 0.05, 3 * 150 + 2, batch)


@pytest.mark.parametrize("rows_per_cn", [8, 9, 15, 17, 40])
def test_short_and_ragged_slices(orc, rows_per_cn):
    """Batch 8: one full batch, one row past it, slices shorter than the 16-row ring and
    than two passes over it, a ragged last slice."""
    c = CONFIGS["F1"]
    K = 5
    n = K * rows_per_cn + 2
    _run(orc, c.layers, c.act, c.init, K, c.lr, n, 8, epochs=2)


@pytest.mark.slow
def test_f1_full_sampled(orc):
    """F1 at its full size (60,000 rows, K = 10, 20 epochs, batch 50; the configuration
    bench.py times) on the resident mini-batch kernel; the oracle re-trains CNs 0 and 9.
    Per-CN rule of tests/cnrule.py (ReLU: a logged kink, R24; the envelope, R22; R34)."""
    from paper_2304_09590_b200 import PNN
    c = CONFIGS["F1"]
    X, y = make_split(c.n_train, "train", 0)
    net = PNN(c.layers, c.act, c.init, c.K, c.lr, seed=0)
    net.set_minibatch(c.batch)
    assert tuple(net.kernel_info()) == (6, 1)
    xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    for _ in range(c.epochs):
        net.train_epoch(xd, yd)
    torch.cuda.synchronize()
    sample = [0, 9]
    okids, _ = orc.train_pnn(c.layers, c.act, c.init, c.K, c.lr, 0, X, y, epochs=c.epochs, batch=c.batch,
                             threads=8, subnets=sample)
    start, count = orc.shard_bounds(c.n_train, c.K)
    from tests.cnrule import cn_bound
    report = []
    for j, i in enumerate(sample):
        kid = net.get_params(i)
        err = float(np.abs(kid - okids[j]).max())
        a, b = int(start[i]), int(start[i] + count[i])
        bound, info = cn_bound(orc, net, c.layers, c.act, c.init, c.lr, X[a:b], y[a:b], err, okids[j], c.epochs,
                               c.batch, kid=kid)
        report.append((i, err, bound, info))
        assert err < TOL or err <= bound, f"CN {i}: max-abs {err:.3g} without a recorded cause: {info}"
    print("F1 full per-CN (index, max-abs, bound, cause):", report)
