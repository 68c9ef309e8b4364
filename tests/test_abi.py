"""The C-ABI library loads and exports every symbol include/pnn.h declares;
host-side validation (no GPU needed: it runs before any CUDA call); the rank
bookkeeping of dist.py agrees with the oracle's slicing.  CPU only."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "pnn.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pnn_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2304_09590_b200 import load
    return load()


def test_every_declared_symbol_is_exported(lib):
    syms = header_symbols()
    assert len(syms) >= 15
    from paper_2304_09590_b200 import EXPORTS
    assert sorted(EXPORTS) == syms
    out = os.popen(f"nm -D --defined-only {os.path.join(ROOT, 'paper_2304_09590_b200', 'libpnn.so')}").read()
    exported = set(re.findall(r" T (pnn_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing


def test_library_is_sm100a(lib):
    out = os.popen("cuobjdump --list-elf "
                   f"{os.path.join(ROOT, 'paper_2304_09590_b200', 'libpnn.so')}").read()
    assert "sm_100a" in out


def _create(lib, layers, act, init=0, K=1, lr=0.1):
    L = np.array(layers, np.int32)
    A = np.array(act, np.int32)
    h = ctypes.c_void_p()
    st = lib.pnn_create(L.ctypes.data_as(ctypes.c_void_p), len(L), A.ctypes.data_as(ctypes.c_void_p),
                        init, K, lr, 0, ctypes.byref(h))
    return st, h, lib.pnn_last_error(None).decode()


def test_create_validation_enumerates_violations(lib):
    # softmax on a hidden layer, zero size, unknown init, K < 1, lr <= 0: all reported at once
    st, h, msg = _create(lib, [784, 0, 10], [3, 3], init=9, K=0, lr=-1.0)
    assert st == 1 and not h.value
    for frag in ("layers[1] = 0", "softmax on hidden layer 1", "init = 9", "n_subnets = 0", "lr"):
        assert frag in msg, (frag, msg)
    st, h, msg = _create(lib, [784], [], K=1)
    assert st == 1 and "n_layers = 1" in msg
    st, h, msg = _create(lib, [784, 10], [7], K=1)
    assert st == 1 and "activation[0] = 7" in msg
    st, h, msg = _create(lib, [784, 10], [0], K=1, lr=float("nan"))
    assert st == 1 and "lr" in msg


def test_null_handle_calls(lib):
    assert lib.pnn_param_count(None) == -1
    assert lib.pnn_destroy(None) == 0
    assert lib.pnn_merge(None, None) == 1
    assert lib.pnn_train_epoch(None, None, None, 0, None) == 1


def test_dist_partition_matches_oracle_slicing(orc):
    from paper_2304_09590_b200.dist import rank_rows, rank_subnets, slice_bounds
    for N, K, G in [(1 << 20, 1024, 8), (60000, 4, 8), (60000, 32, 8), (1003, 7, 3), (10, 4, 2)]:
        start, count = orc.shard_bounds(N, K)
        for i in range(K):
            assert slice_bounds(N, K, i) == (start[i], count[i])
        covered = 0
        for r in range(G):
            f, c = rank_subnets(K, G, r)
            s, n = rank_rows(N, K, G, r)
            assert s == covered
            covered += n
            if c:
                # the library splits a rank's rows among its CNs by R17 again: same slices
                loc_s, loc_c = orc.shard_bounds(n, c)
                np.testing.assert_array_equal(loc_s + s, start[f:f + c])
                np.testing.assert_array_equal(loc_c, count[f:f + c])
        assert covered == N
