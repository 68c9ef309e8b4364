"""The tcgen05 GEMM of the bf16 mini-batch variant (a10) against torch:
C[z] = A[z] · B[z]ᵀ with bf16 operands and fp32 accumulation, on the shapes the
C5 step uses (K = 784 with a ragged last K tile, K = 64, K = 1024, N = 784 with a
ragged last N tile).  Marked gpu."""
import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2304_09590_b200 import load
    L = load()
    L.pnn_debug_tc_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5
    L.pnn_debug_tc_gemm.restype = ctypes.c_int
    return L


@pytest.mark.parametrize("Z,M,N,K,bn", [
    (2, 256, 64, 784, 64),
    (1, 128, 256, 64, 256),
    (3, 1024, 784, 64, 256),
    (2, 128, 128, 1024, 128),
    (8, 1024, 64, 1024, 64),
])
def test_tc_gemm_matches_torch(lib, Z, M, N, K, bn):
    g = torch.Generator(device="cuda").manual_seed(Z * 1000 + K)
    A = torch.randn(Z, M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(Z, N, K, device="cuda", generator=g).to(torch.bfloat16)
    C = torch.full((Z, M, N), float("nan"), device="cuda")
    rc = lib.pnn_debug_tc_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), Z, M, N, K, bn)
    assert rc == 0, rc
    ref = torch.bmm(A.double(), B.double().transpose(1, 2)).float()
    err = (C - ref).abs().max().item()
    assert err < 1e-3 * K ** 0.5, err
