"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the
same seeded inputs.  Marked gpu; run on a B200 via gpurun.

Tolerances (BASELINE.json north_star; DESIGN.md §3 R22/R24/R26):
  * fp32 per-sample SGD: every weight and bias of every CN, and of the merged
    network, within max-abs 1e-4 of the fp32 oracle after the epoch(s);
  * merge of the GPU's own children: bit-exact vs the oracle's merge (both sum
    in fp64 in ascending CN order, divide by K, round once);
  * predicted labels: bit-exact vs the oracle's fp64 readout of the same weights;
  * init: bit-exact (both sides implement the R15 counter-based generator).
"""
import numpy as np
import pytest
import torch

from datagen import make_rows, make_split
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


def PNN(*a, kernel="auto", **k):
    from paper_2304_09590_b200 import PNN as _P
    net = _P(*a, **k)
    net.set_kernel(kernel)
    return net


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


KERNELS = ["reference", "auto"]


def _train(cfg_layers, act, init, K, lr, X, y, epochs=1, kernel="auto", batch=1, variant=None):
    net = PNN(cfg_layers, act, init, K, lr, seed=0, kernel=kernel)
    if batch > 1:
        net.set_minibatch(batch)
    if variant is not None:
        net.set_variant(variant)
    xd, yd = dev(X), dev(y)
    for _ in range(epochs):
        net.train_epoch(xd, yd)
    net.merge()
    torch.cuda.synchronize()
    kids = np.stack([net.get_params(i) for i in range(K)])
    return net, kids, net.get_params(-1)


@pytest.mark.parametrize("init", ["normal", "uniform", "xavier", "he"])
def test_init_bit_exact_and_cloned(orc, init):
    layers = [784, 37, 10]
    net = PNN(layers, ["tanh", "softmax"], init, 3, 0.1, seed=1234)
    ref = orc.init_params(layers, init, 1234)
    np.testing.assert_array_equal(net.get_params(-1), ref)
    for i in range(3):
        np.testing.assert_array_equal(net.get_params(i), ref)
    # merge of untrained clones == init exactly (R18)
    net.merge()
    np.testing.assert_array_equal(net.get_params(-1), ref)


@pytest.mark.parametrize("kernel", KERNELS)
def test_c1_full(orc, kernel):
    """configs[0] at full size: 1 CN, 784-16-10 sigmoid, U[-.5,.5], η=0.1, 1000 rows."""
    c = CONFIGS["C1"]
    X, y = make_split(c.n_train, "train", 0)
    Xt, _ = make_split(c.n_test, "test", 0)
    net, kids, merged = _train(c.layers, c.act, c.init, c.K, c.lr, X, y, kernel=kernel)
    okids, omerged = orc.train_pnn(c.layers, c.act, c.init, c.K, c.lr, 0, X, y)
    assert np.abs(kids - okids).max() < TOL
    assert np.abs(merged - omerged).max() < TOL
    np.testing.assert_array_equal(merged, kids[0])            # K = 1: merge is the identity
    lab = net.predict(dev(Xt)).cpu().numpy()
    np.testing.assert_array_equal(lab, orc.predict(c.layers, c.act, merged, Xt))
    # labels of the GPU-trained vs the oracle-trained network
    assert (orc.predict(c.layers, c.act, omerged, Xt) != lab).sum() == 0


REDUCED = [  # (config, K, rows, epochs): several CNs, a ragged row count
    ("C2", 4, 4 * 700 + 3, 1),
    ("C3", 8, 8 * 120 + 5, 2),
    ("C4", 64, 64 * 96 + 37, 1),
]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("name,K,n,epochs", REDUCED)
def test_reduced_configs(orc, name, K, n, epochs, kernel):
    c = CONFIGS[name]
    X, y = make_split(n, "train", 0)
    Xt, _ = make_split(500, "test", 0)
    net, kids, merged = _train(c.layers, c.act, c.init, K, c.lr, X, y, epochs, kernel)
    okids, omerged = orc.train_pnn(c.layers, c.act, c.init, K, c.lr, 0, X, y, epochs=epochs, threads=8)
    err = np.abs(kids - okids).max(axis=1)
    assert err.max() < TOL, f"per-CN max-abs {err}"
    assert np.abs(merged - omerged).max() < TOL
    np.testing.assert_array_equal(merged, orc.merge(kids))    # merge arithmetic: bit-exact
    lab = net.predict(dev(Xt)).cpu().numpy()
    np.testing.assert_array_equal(lab, orc.predict(c.layers, c.act, merged, Xt))
    lab0 = net.predict(dev(Xt), subnet=0).cpu().numpy()
    np.testing.assert_array_equal(lab0, orc.predict(c.layers, c.act, kids[0], Xt))


@pytest.mark.parametrize("kernel", KERNELS)
def test_leaky_relu_c4_shape(orc, kernel):
    """f3: leaky ReLU hidden layer (slope 0.01, R30) on the C4 shape,
    reference and resident kernels vs the oracle."""
    c = CONFIGS["C4"]
    act = ["leaky_relu", "softmax"]
    K, n = 32, 32 * 80 + 11
    X, y = make_split(n, "train", 0)
    Xt, _ = make_split(500, "test", 0)
    net, kids, merged = _train(c.layers, act, c.init, K, c.lr, X, y, 1, kernel)
    if kernel == "auto":
        assert net.kernel_info()[0] == 2                       # the resident kernel took it
    okids, omerged = orc.train_pnn(c.layers, act, c.init, K, c.lr, 0, X, y, threads=8)
    assert np.abs(kids - okids).max() < TOL
    assert np.abs(merged - omerged).max() < TOL
    lab = net.predict(dev(Xt)).cpu().numpy()
    np.testing.assert_array_equal(lab, orc.predict(c.layers, act, merged, Xt))


def test_evaluate_matches_oracle(orc):
    """f2 metrics (accuracy, confidence, cost; R29) of the merged net and of single
    CNs, on the GPU's own trained parameters, vs the oracle's fp64 definitions."""
    c = CONFIGS["C4"]
    K = 8
    X, y = make_split(K * 200, "train", 0)
    Xt, yt = make_split(1003, "test", 0)
    net, kids, merged = _train(c.layers, c.act, c.init, K, c.lr, X, y)
    for sub, p in [(-1, merged), (0, kids[0]), (5, kids[5])]:
        got = net.evaluate(dev(Xt), dev(yt), subnet=sub)
        ref = orc.evaluate(c.layers, c.act, p, Xt, yt)
        assert got[0] == ref[0]
        np.testing.assert_allclose(got[1:], ref[1:], rtol=1e-12)
    # sigmoid output (C2 shape): confidence / cost from φ_L
    c2 = CONFIGS["C2"]
    net2 = PNN(c2.layers, c2.act, c2.init, 1, c2.lr, seed=3)
    got = net2.evaluate(dev(Xt), dev(yt))
    ref = orc.evaluate(c2.layers, c2.act, net2.get_params(-1), Xt, yt)
    assert got[0] == ref[0]
    np.testing.assert_allclose(got[1:], ref[1:], rtol=1e-12)


@pytest.mark.parametrize("kernel", KERNELS)
def test_slots_do_not_change_results(kernel):
    """f4: training in waves of `slots` CNs gives bit-identical CNs."""
    c = CONFIGS["C4"]
    K = 12
    X, y = make_split(K * 40 + 5, "train", 0)
    outs = []
    for slots in (0, 1, 5):
        net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0, kernel=kernel)
        net.set_slots(slots)
        net.train_epoch(dev(X), dev(y))
        torch.cuda.synchronize()
        outs.append(np.stack([net.get_params(i) for i in range(K)]))
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])


@pytest.mark.parametrize("name,K,n,epochs", REDUCED + [("C1", 2, 2 * 300 + 1, 1)])
def test_cluster_kernel(orc, name, K, n, epochs):
    """The cluster kernel (weights in the shared memory of a cluster of CTAs, any
    depth; AUTO's choice for C3) forced on every config shape, vs the oracle."""
    c = CONFIGS[name]
    X, y = make_split(n, "train", 0)
    net, kids, merged = _train(c.layers, c.act, c.init, K, c.lr, X, y, epochs, "cluster")
    assert net.kernel_info()[0] == 5
    okids, omerged = orc.train_pnn(c.layers, c.act, c.init, K, c.lr, 0, X, y, epochs=epochs, threads=8)
    err = np.abs(kids - okids).max(axis=1)
    assert err.max() < TOL, f"per-CN max-abs {err}"
    assert np.abs(merged - omerged).max() < TOL


@pytest.mark.parametrize("kernel", ["resident", "v8", "tmem", "ws", "cluster", "reference"])
@pytest.mark.parametrize("rows_per_cn", [1, 2, 3, 4, 5, 6, 17])
def test_short_slices(orc, kernel, rows_per_cn):
    """Slices shorter than the resident kernels' lookahead / prefetch depths (L = 4,
    8 rows in flight) and the cluster kernel's ring, with one ragged slice.  6 CNs fit
    the GPU, so AUTO's resident plan is v10; v8 / tmem / ws force those variants."""
    variant = None
    if kernel in ("v8", "tmem", "ws"):
        variant, kernel = kernel, "resident"
    c = CONFIGS["C4"]
    K = 6
    n = K * rows_per_cn + (1 if rows_per_cn > 1 else 0)
    X, y = make_split(n, "train", 0)
    _, kids, merged = _train(c.layers, c.act, c.init, K, c.lr, X, y, 2, kernel, variant=variant)
    okids, omerged = orc.train_pnn(c.layers, c.act, c.init, K, c.lr, 0, X, y, epochs=2)
    assert np.abs(kids - okids).max() < TOL
    assert np.abs(merged - omerged).max() < TOL


def test_resident_v10_split_variant(orc):
    """The v10 resident variant (chain on a dedicated CTA of a 3-CTA cluster) on the C4
    and C2 shapes with ragged and short slices."""
    for name, K, n in [("C4", 16, 16 * 70 + 5), ("C2", 4, 4 * 300 + 3), ("C4", 6, 6 * 3 + 1)]:
        c = CONFIGS[name]
        X, y = make_split(n, "train", 0)
        net, kids, merged = _train(c.layers, c.act, c.init, K, c.lr, X, y, 1, "resident", variant="v10")
        assert net.kernel_variant() == 10
        okids, omerged = orc.train_pnn(c.layers, c.act, c.init, K, c.lr, 0, X, y, threads=8)
        assert np.abs(kids - okids).max() < TOL, name
        assert np.abs(merged - omerged).max() < TOL, name


TMEM_CASES = [  # (config, activations, K, rows): C4 ragged, C2 (H = 100, sigmoid/½-SSE), every pair
    ("C4", None, 40, 40 * 90 + 7),
    ("C2", None, 4, 4 * 400 + 3),
    ("C4", ["tanh", "softmax"], 8, 8 * 60 + 1),
    ("C4", ["sigmoid", "softmax"], 8, 8 * 60 + 1),
    ("C4", ["tanh", "tanh"], 8, 8 * 60 + 1),
    ("C4", ["relu", "sigmoid"], 8, 8 * 60 + 1),
    ("C4", ["leaky_relu", "softmax"], 8, 8 * 60 + 1),
]


@pytest.mark.parametrize("name,act,K,n", TMEM_CASES)
def test_resident_tmem_variant(orc, name, act, K, n):
    """The TMEM resident variant (v11, k_tmem.cu: one SM per CN, W1 rows in registers
    and tensor memory, the R27 Gram terms formed in the launch) vs the oracle."""
    c = CONFIGS[name]
    act = act or c.act
    X, y = make_split(n, "train", 0)
    net, kids, merged = _train(c.layers, act, c.init, K, c.lr, X, y, 1, "resident", variant="tmem")
    assert net.kernel_variant() == 11 and net.kernel_info() == (2, 1)
    okids, omerged = orc.train_pnn(c.layers, act, c.init, K, c.lr, 0, X, y, threads=8)
    err = np.abs(kids - okids).max(axis=1)
    assert err.max() < TOL, f"per-CN max-abs {err}"
    assert np.abs(merged - omerged).max() < TOL


@pytest.mark.parametrize("name,act,K,n", TMEM_CASES)
def test_resident_ws_variant(orc, name, act, K, n):
    """The warp-specialised TMEM variant (v12, k_ws.cu: v11's W1 placement plus one row per
    warp in shared memory, the per-sample chain on its own warpgroup) vs the oracle."""
    c = CONFIGS[name]
    act = act or c.act
    X, y = make_split(n, "train", 0)
    net, kids, merged = _train(c.layers, act, c.init, K, c.lr, X, y, 1, "resident", variant="ws")
    assert net.kernel_variant() == 12 and net.kernel_info()[0] == 2
    okids, omerged = orc.train_pnn(c.layers, act, c.init, K, c.lr, 0, X, y, threads=8)
    err = np.abs(kids - okids).max(axis=1)
    assert err.max() < TOL, f"per-CN max-abs {err}"
    assert np.abs(merged - omerged).max() < TOL


def test_kernel_timing_hook():
    """pnn_kernel_timing brackets each training-kernel launch with CUDA events."""
    c = CONFIGS["C4"]
    X, y = make_split(16 * 40, "train", 0)
    net = PNN(c.layers, c.act, c.init, 16, c.lr, seed=0)
    net.kernel_timing(True)
    for _ in range(3):
        net.train_epoch(dev(X), dev(y))
    ms, n = net.kernel_timing(False)
    assert n == 3 and ms > 0.0
    net.train_epoch(dev(X), dev(y))          # stopped: nothing recorded
    assert net.kernel_timing(False) == (0.0, 0)


def test_determinism_and_kernel_agreement(orc):
    c = CONFIGS["C4"]
    X, y = make_split(32 * 64, "train", 0)
    runs = [_train(c.layers, c.act, c.init, 32, c.lr, X, y)[1] for _ in range(2)]
    np.testing.assert_array_equal(runs[0], runs[1])                 # bit-identical reruns


def test_host_input_path_matches_device_path():
    c = CONFIGS["C4"]
    X, y = make_split(16 * 50 + 3, "train", 0)
    a = _train(c.layers, c.act, c.init, 16, c.lr, X, y)[1]
    net = PNN(c.layers, c.act, c.init, 16, c.lr, seed=0)
    net.train_epoch_host(torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory())
    torch.cuda.synchronize()
    b = np.stack([net.get_params(i) for i in range(16)])
    np.testing.assert_array_equal(a, b)


def test_host_input_back_to_back_calls():
    """Host-input calls issued back to back with different data: each group's staging rows are
    overwritten only after the previous call's launch that reads them (per-group release when
    the grouping repeats, a full wait when it changes) — same bits as the device path."""
    c = CONFIGS["C4"]
    K = 300                                          # 3 waves of 148 CNs: 3 host-copy groups
    sets = [make_split(K * 12 + 7, "train", s) for s in (0, 1, 2)] + [make_split(K * 9 + 1, "train", 3)]
    ref = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
    for X, y in sets:
        ref.train_epoch(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
    net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
    pinned = [(torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory()) for X, y in sets]
    for xh, yh in pinned:
        net.train_epoch_host(xh, yh)
    torch.cuda.synchronize()
    for i in (0, 1, 147, 148, 299):
        np.testing.assert_array_equal(net.get_params(i), ref.get_params(i))


def test_k1_is_snn_and_duplicated_shards(orc):
    """K=1 handle == the sequential network; K CNs on K identical slices stay
    identical and merge back to any one of them (R18)."""
    c = CONFIGS["C1"]
    X, y = make_split(200, "train", 0)
    _, kids, merged = _train(c.layers, c.act, c.init, 4, c.lr, np.tile(X[:50], (4, 1)), np.tile(y[:50], 4))
    for k in kids:
        np.testing.assert_array_equal(k, kids[0])
    np.testing.assert_array_equal(merged, kids[0])


# (kernel, variant, expected kernel id): reference; AUTO = the persistent resident mini-batch
# kernel (6); the mb_step variant = the fp32 step kernels (4)
MB_KERNELS = [("reference", None, 1), ("auto", None, 6), ("auto", "mb_step", 4)]


@pytest.mark.parametrize("kernel,mbres,kid", MB_KERNELS)
def test_minibatch_fp32(orc, kernel, mbres, kid):
    """Mini-batch GD, B=8 with a short last batch (R14), on the
    reference kernel, the resident mini-batch kernel and the fp32 step kernels."""
    c = CONFIGS["C4"]
    X, y = make_split(4 * 61, "train", 0)
    net, kids, merged = _train(c.layers, c.act, c.init, 4, c.lr, X, y, batch=8, kernel=kernel, variant=mbres)
    assert net.kernel_info()[0] == kid
    okids, omerged = orc.train_pnn(c.layers, c.act, c.init, 4, c.lr, 0, X, y, batch=8)
    assert np.abs(kids - okids).max() < TOL
    assert np.abs(merged - omerged).max() < TOL


@pytest.mark.parametrize("kernel,mbres,kid", MB_KERNELS)
def test_f1_paper_workload_reduced(orc, kernel, mbres, kid):
    """f1: the paper's own setting (784-256-10 ReLU/softmax, N(0,1) init, fp32
    mini-batch B=50, η 0.1) on 3 CNs with ragged
    slices and a short last batch, 2 epochs, vs the oracle."""
    c = CONFIGS["F1"]
    K, n = 3, 3 * (50 * 3 + 17) + 2
    X, y = make_split(n, "train", 0)
    net, kids, merged = _train(c.layers, c.act, c.init, K, c.lr, X, y, epochs=2, batch=c.batch, kernel=kernel,
                               variant=mbres)
    assert net.kernel_info()[0] == kid
    okids, omerged = orc.train_pnn(c.layers, c.act, c.init, K, c.lr, 0, X, y, epochs=2, batch=c.batch,
                                   threads=K)
    from tests.cnrule import check_cns, check_merged
    bounds = check_cns(orc, net, c.layers, c.act, c.init, K, c.lr, X, y, kids, okids, 2, c.batch)
    check_merged(merged, omerged, bounds)


def test_error_paths():
    from paper_2304_09590_b200 import PnnError
    c = CONFIGS["C4"]
    net = PNN(c.layers, c.act, c.init, 8, c.lr)
    X, y = make_split(5, "train", 0)
    with pytest.raises(PnnError) as e:
        net.train_epoch(dev(X), dev(y))                     # 5 rows < 8 CNs
    assert e.value.status == 3
    with pytest.raises(PnnError) as e:
        net.get_params(8)
    assert e.value.status == 1
    with pytest.raises(PnnError) as e:
        net.set_params(np.zeros(10, np.float32))
    assert e.value.status == 2
    net.set_minibatch(4)
    with pytest.raises(PnnError) as e:
        net.train_epoch(dev(np.tile(X, (4, 1))), dev(np.tile(y, 4)))   # 20 rows: slice 2 < batch 4
    assert e.value.status == 3
    with pytest.raises(PnnError) as e:
        net.set_slots(-1)
    assert e.value.status == 1
    Xt, yt = make_split(16, "test", 0)
    with pytest.raises(PnnError) as e:
        net.evaluate(dev(Xt[:0]), dev(yt[:0]))              # n = 0
    assert e.value.status == 1
    with pytest.raises(PnnError) as e:
        net.evaluate(dev(Xt), dev(yt), subnet=8)            # not a local CN
    assert e.value.status == 1
    with pytest.raises(PnnError) as e:
        net.set_kernel(3)                                   # PNN_KERNEL_TC_BF16: not settable
    assert e.value.status == 1
    # the handle is still usable after validation errors
    X, y = make_split(64, "train", 0)
    net.train_epoch(dev(X), dev(y))
    torch.cuda.synchronize()
    acc, conf, cost = net.evaluate(dev(Xt), dev(yt), subnet=0)
    assert 0.0 <= acc <= 1.0 and 0.1 <= conf <= 1.0 and cost >= 0.0


def test_set_params_roundtrip_and_predict_subnet(orc):
    c = CONFIGS["C4"]
    net = PNN(c.layers, c.act, c.init, 4, c.lr)
    rng = np.random.default_rng(0)
    p = rng.normal(size=net.param_count).astype(np.float32)
    net.set_params(p, subnet=2)
    np.testing.assert_array_equal(net.get_params(2), p)
    Xt, _ = make_split(300, "test", 0)
    lab = net.predict(dev(Xt), subnet=2).cpu().numpy()
    np.testing.assert_array_equal(lab, orc.predict(c.layers, c.act, p, Xt))
    net.set_params(p, subnet=-2)
    np.testing.assert_array_equal(net.get_params(-1), p)


# Full-size, full-population parity (every CN of C1-C5 vs the oracle, merged nets, R24
# kink accounting, full-test-set labels): tests/test_gpu_fullsize.py.


@pytest.mark.parametrize("name,K,rows,batch", [
    ("C3", 40, 40 * 12 + 5, 1),      # deep cluster variant, 2 host-copy groups (18 CNs per group)
    ("F1", 40, 40 * 60 + 7, 50),     # resident mini-batch kernel, 2 groups
    ("C2", 4, 4 * 100 + 3, 1),       # v10 resident variant
])
def test_host_input_path_other_kernels(name, K, rows, batch):
    """pnn_train_epoch_host (H2D copies pipelined with training in CN groups) gives the
    device path's parameters bit for bit on the deep, mini-batch and v10 kernels."""
    c = CONFIGS[name]
    X, y = make_split(rows, "train", 0)
    a = _train(c.layers, c.act, c.init, K, c.lr, X, y, batch=batch)[1]
    net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
    if batch > 1:
        net.set_minibatch(batch)
    net.train_epoch_host(torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory())
    torch.cuda.synchronize()
    b = np.stack([net.get_params(i) for i in range(K)])
    np.testing.assert_array_equal(a, b)
