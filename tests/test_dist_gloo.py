"""The N>1 path's host logic on CPU: world_size-2 gloo processes.

Each rank takes exactly the CNs and rows `paper_2304_09590_b200.dist` assigns
(PAPER.md:166-169 slicing, R17), trains them (oracle, CPU), sums its children
in fp64, all-reduces the partial sums (the same reduction pnn_merge performs
with ncclAllReduce over NVLink), divides by K and rounds once (R18).  The
result must equal the single-process merge of all children, and every CN
must be bit-identical to its single-process training (placement invariance).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from datagen import make_rows, make_split

LAYERS, ACT, INIT, LR = [784, 24, 10], ["relu", "softmax"], "he", 0.01


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, K, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2304_09590_b200.dist import rank_rows, rank_subnets
    first, cnt = rank_subnets(K, world, rank)
    r0, nrows = rank_rows(N, K, world, rank)
    X, y = make_rows(r0, nrows, "train", 0)
    p0 = oracle.init_params(LAYERS, INIT, 0)
    # the library's local split: R17 again over this rank's rows
    ls, lc = oracle.shard_bounds(nrows, cnt) if cnt else (np.zeros(0, int), np.zeros(0, int))
    kids = [oracle.train(LAYERS, ACT, p0, X[s:s + c], y[s:s + c], LR) for s, c in zip(ls, lc)]
    psum = np.zeros(p0.size, dtype=np.float64)
    for k in kids:
        psum += k.astype(np.float64)
    t = torch.from_numpy(psum)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    merged = (t.numpy() / K).astype(np.float32)
    np.save(os.path.join(out_dir, f"merged{rank}.npy"), merged)
    np.save(os.path.join(out_dir, f"kids{rank}.npy"), np.stack(kids) if kids else np.zeros((0, p0.size), np.float32))
    dist.destroy_process_group()


@pytest.mark.parametrize("N,K", [(8 * 40, 8), (7 * 31 + 5, 7), (3 * 50, 3)])
def test_two_rank_merge_equals_single_process(orc, tmp_path, N, K):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), N, K, str(tmp_path)), nprocs=world, join=True)
    X, y = make_split(N, "train", 0)
    kids, merged = orc.train_pnn(LAYERS, ACT, INIT, K, LR, 0, X, y)
    m0 = np.load(tmp_path / "merged0.npy")
    m1 = np.load(tmp_path / "merged1.npy")
    np.testing.assert_array_equal(m0, m1)                       # every rank holds the merged net
    assert np.abs(m0 - merged).max() <= 1e-7                     # fp64 sums: equal up to final rounding
    rk = np.concatenate([np.load(tmp_path / "kids0.npy"), np.load(tmp_path / "kids1.npy")])
    np.testing.assert_array_equal(rk, kids)                     # placement invariance, bit-exact
