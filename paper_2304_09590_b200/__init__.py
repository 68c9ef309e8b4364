"""B200-native PNN hot path (arXiv 2304.09590): per-sample backprop SGD of many
independent child networks + averaging merge, behind the C ABI include/pnn.h.

The package holds only what the path needs: csrc/ (CUDA kernels + the C ABI,
built into libpnn.so), the ctypes binding (pnn.py) and the rank bookkeeping for
torch.distributed launches (dist.py).
"""
from .pnn import (PNN, PnnError, load, EXPORTS, ACT, INIT, KERNEL, PNN_FP32, PNN_BF16,
                  PNN_KERNEL_AUTO, PNN_KERNEL_REFERENCE, PNN_KERNEL_RESIDENT, LIB_PATH)

__all__ = ["PNN", "PnnError", "load", "EXPORTS", "ACT", "INIT", "KERNEL", "PNN_FP32", "PNN_BF16",
           "PNN_KERNEL_AUTO", "PNN_KERNEL_REFERENCE", "PNN_KERNEL_RESIDENT", "LIB_PATH"]
