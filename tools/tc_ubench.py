"""Standalone timings of the tcgen05 GEMM (EPI_STORE_F32 epilogue) at the C5 step shapes,
for ncu (tools only):  ncu --cache-control none --metrics gpu__time_duration.sum python tools/tc_ubench.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_09590_b200 import load
L = load()
L.pnn_debug_tc_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5
shapes = [("F1", 8, 1024, 64, 784, 64), ("F2", 8, 1024, 64, 1024, 64), ("B5", 8, 1024, 784, 64, 256),
          ("B3", 8, 1024, 1024, 64, 256)]
for name, Z, M, N, K, bn in shapes:
    A = torch.randn(Z, M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(Z, N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(Z, M, N, device="cuda")
    for _ in range(3):
        assert L.pnn_debug_tc_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), Z, M, N, K, bn) == 0
    print(name, "ok")
