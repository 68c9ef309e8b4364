"""The library's multi-rank path on one GPU (PAPER.md:156 SPMD,
:166-172 and :233-238 slices then averaging), through the C ABI.

NCCL cannot put two ranks of one communicator on one GPU, so the ranks here are
handles made with pnn_set_comm(nranks, rank, id = NULL): the library does its rank
bookkeeping (owned CNs, pnn_local_rows) and the two device steps of the merge
(pnn_merge_partial: fp64 sum of the rank's CNs in ascending order; pnn_merge_finish:
÷K and one rounding) exactly as pnn_merge does around its ncclAllReduce; the test
plays the all-reduce by adding the ranks' fp64 partial sums.  Checked: every CN is
bit-identical for every rank split (no data moves between ranks), idle ranks (K < G)
train nothing and contribute zeros, and the multi-rank merge equals the single-rank
merge (fp64 sums of fp32 values: the split changes no bit of the rounded result here).
"""
import numpy as np
import pytest
import torch

from datagen import make_split
from workloads import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _single(c, K, X, y):
    from paper_2304_09590_b200 import PNN
    net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
    net.train_epoch(dev(X), dev(y))
    net.merge()
    torch.cuda.synchronize()
    return np.stack([net.get_params(i) for i in range(K)]), net.get_params(-1)


@pytest.mark.parametrize("K,G", [(8, 2), (3, 2), (1, 2), (5, 4), (2, 4)])
def test_ranks_train_their_slices_and_merge(orc, K, G):
    from paper_2304_09590_b200 import PNN, PnnError
    from paper_2304_09590_b200.dist import rank_rows, rank_subnets
    c = CONFIGS["C4"]
    N = K * 70 + 3
    X, y = make_split(N, "train", 0)
    kids_ref, merged_ref = _single(c, K, X, y)
    nets, sums = [], []
    for r in range(G):
        net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
        net.set_comm(G, r, None)
        first, count = net.local_subnets()
        assert (first, count) == rank_subnets(K, G, r)
        r0, nr = net.local_rows(N)
        assert (r0, nr) == rank_rows(N, K, G, r)
        if count == 0:                               # idle rank: no rows, no pointers
            assert nr == 0
            net.train_epoch(None, None)
        else:
            net.train_epoch(dev(X[r0:r0 + nr]), dev(y[r0:r0 + nr]))
        s = torch.empty(net.param_count, dtype=torch.float64, device="cuda")
        net.merge_partial(s)
        with pytest.raises(PnnError) as e:           # no communicator: pnn_merge refuses
            net.merge()
        assert e.value.status == 4
        torch.cuda.synchronize()
        for i in range(first, first + count):        # CNs bit-identical for every split
            np.testing.assert_array_equal(net.get_params(i), kids_ref[i])
        if count == 0:
            assert torch.count_nonzero(s).item() == 0  # an idle rank contributes zeros
        nets.append(net)
        sums.append(s)
    total = sums[0].clone()
    for s in sums[1:]:
        total += s                                   # the all-reduce
    for net in nets:
        net.merge_finish(total)
    torch.cuda.synchronize()
    for net in nets:
        m = net.get_params(-1)
        np.testing.assert_array_equal(m, merged_ref)
        np.testing.assert_array_equal(m, orc.merge(kids_ref))


def test_partial_finish_equals_merge():
    """merge_sum → merge_finish on one rank == the fused single-rank merge, bit for bit."""
    from paper_2304_09590_b200 import PNN
    c = CONFIGS["C4"]
    X, y = make_split(16 * 40, "train", 0)
    net = PNN(c.layers, c.act, c.init, 16, c.lr, seed=0)
    net.train_epoch(dev(X), dev(y))
    net.merge()
    torch.cuda.synchronize()
    a = net.get_params(-1)
    s = torch.empty(net.param_count, dtype=torch.float64, device="cuda")
    net.merge_partial(s)
    net.merge_finish(s)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(net.get_params(-1), a)


def test_idle_rank_rejects_rows():
    from paper_2304_09590_b200 import PNN, PnnError
    c = CONFIGS["C4"]
    net = PNN(c.layers, c.act, c.init, 1, c.lr, seed=0)
    net.set_comm(2, 0, None)                         # K = 1 < G = 2: rank 0 owns no CN
    assert net.local_subnets() == (0, 0)
    X, y = make_split(8, "train", 0)
    with pytest.raises(PnnError) as e:
        net.train_epoch(dev(X), dev(y))
    assert e.value.status == 3


def test_one_rank_nccl_merge():
    """pnn_set_comm(1, 0, id) makes a real one-rank NCCL communicator: pnn_merge then runs
    the multi-rank chain (fp64 partial sum → ncclAllReduce → ÷K, one rounding) on hardware,
    and must equal the fused local merge and the oracle's merge bit for bit (R18)."""
    from paper_2304_09590_b200 import PNN
    from paper_2304_09590_b200.dist import nccl_unique_id_bytes
    c = CONFIGS["C4"]
    K = 6
    X, y = make_split(K * 50 + 5, "train", 0)
    kids_ref, merged_ref = _single(c, K, X, y)
    net = PNN(c.layers, c.act, c.init, K, c.lr, seed=0)
    net.set_comm(1, 0, nccl_unique_id_bytes(0))
    assert net.local_subnets() == (0, K)
    net.train_epoch(dev(X), dev(y))
    net.merge()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(net.get_params(-1), merged_ref)
    net.close()
