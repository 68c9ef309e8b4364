"""Thin ctypes binding of include/pnn.h (argument marshalling only).

Every step of the hot path runs in libpnn.so's CUDA kernels; there is no CPU
or PyTorch fallback — a missing library raises at import of this module's
first call.  torch is used only for device memory (tensors), streams and
process groups.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpnn.so")

PNN_OK, PNN_ERR_INVALID, PNN_ERR_SHAPE, PNN_ERR_DATA, PNN_ERR_STATE, PNN_ERR_CUDA, \
    PNN_ERR_NCCL, PNN_ERR_OOM = range(8)
STATUS_NAMES = ["PNN_OK", "PNN_ERR_INVALID", "PNN_ERR_SHAPE", "PNN_ERR_DATA", "PNN_ERR_STATE",
                "PNN_ERR_CUDA", "PNN_ERR_NCCL", "PNN_ERR_OOM"]
PNN_SIGMOID, PNN_TANH, PNN_RELU, PNN_SOFTMAX, PNN_LEAKY_RELU = 0, 1, 2, 3, 4
PNN_INIT_NORMAL, PNN_INIT_UNIFORM, PNN_INIT_XAVIER_NORMAL, PNN_INIT_HE_NORMAL = 0, 1, 2, 3
PNN_FP32, PNN_BF16 = 0, 1
PNN_KERNEL_AUTO, PNN_KERNEL_REFERENCE, PNN_KERNEL_RESIDENT, PNN_KERNEL_TC_BF16, PNN_KERNEL_MB_F32, \
    PNN_KERNEL_CLUSTER, PNN_KERNEL_MB_RESIDENT = 0, 1, 2, 3, 4, 5, 6
PNN_VARIANT_AUTO, PNN_VARIANT_RESIDENT_V8, PNN_VARIANT_RESIDENT_V10, PNN_VARIANT_RESIDENT_TMEM = 0, 8, 10, 11
PNN_VARIANT_RESIDENT_WS = 12
PNN_VARIANT_CLUSTER_GENERIC, PNN_VARIANT_CLUSTER_DEEP, PNN_VARIANT_MB_STEP, PNN_VARIANT_MB_RESIDENT = 20, 21, 30, 31
VARIANT = {"auto": PNN_VARIANT_AUTO, "v8": PNN_VARIANT_RESIDENT_V8, "v10": PNN_VARIANT_RESIDENT_V10,
             "tmem": PNN_VARIANT_RESIDENT_TMEM, "ws": PNN_VARIANT_RESIDENT_WS, "cluster": PNN_VARIANT_CLUSTER_GENERIC, "deep": PNN_VARIANT_CLUSTER_DEEP,
           "mb_step": PNN_VARIANT_MB_STEP, "mb_resident": PNN_VARIANT_MB_RESIDENT}
ACT = {"sigmoid": PNN_SIGMOID, "tanh": PNN_TANH, "relu": PNN_RELU, "softmax": PNN_SOFTMAX,
       "leaky_relu": PNN_LEAKY_RELU}
INIT = {"normal": PNN_INIT_NORMAL, "uniform": PNN_INIT_UNIFORM, "xavier": PNN_INIT_XAVIER_NORMAL,
        "he": PNN_INIT_HE_NORMAL}
KERNEL = {"auto": PNN_KERNEL_AUTO, "reference": PNN_KERNEL_REFERENCE, "resident": PNN_KERNEL_RESIDENT,
          "cluster": PNN_KERNEL_CLUSTER}

EXPORTS = ["pnn_create", "pnn_set_comm", "pnn_set_minibatch", "pnn_set_kernel", "pnn_train_epoch",
           "pnn_train_epoch_host", "pnn_merge", "pnn_predict", "pnn_get_params", "pnn_set_params",
           "pnn_device_params", "pnn_param_count", "pnn_local_subnets", "pnn_kernel_info",
           "pnn_last_error", "pnn_destroy", "pnn_evaluate", "pnn_set_slots", "pnn_kernel_timing",
           "pnn_set_variant", "pnn_kernel_variant", "pnn_local_rows", "pnn_merge_partial", "pnn_merge_finish"]

_lib = None


class PnnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


def load(path: str | None = None):
    """Load libpnn.so (or $PNN_LIB, an experiment variant) and declare every
    signature of include/pnn.h."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PNN_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    V, I32, I64, F, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_uint64
    P32 = ctypes.POINTER(ctypes.c_int32)
    sig = {
        "pnn_create": ([V, I32, V, I32, I32, F, U64, ctypes.POINTER(V)], I32),
        "pnn_set_comm": ([V, V, I32, I32], I32),
        "pnn_set_minibatch": ([V, I32, I32], I32),
        "pnn_set_kernel": ([V, I32], I32),
        "pnn_train_epoch": ([V, V, V, I64, V], I32),
        "pnn_train_epoch_host": ([V, V, V, I64, V], I32),
        "pnn_merge": ([V, V], I32),
        "pnn_predict": ([V, I32, V, I64, V, V], I32),
        "pnn_get_params": ([V, I32, V, I64], I32),
        "pnn_set_params": ([V, I32, V, I64], I32),
        "pnn_device_params": ([V, I32], V),
        "pnn_param_count": ([V], I64),
        "pnn_local_subnets": ([V, P32, P32], I32),
        "pnn_kernel_info": ([V, P32, P32], I32),
        "pnn_last_error": ([V], ctypes.c_char_p),
        "pnn_destroy": ([V], I32),
        "pnn_evaluate": ([V, I32, V, V, I64, V, V], I32),
        "pnn_set_slots": ([V, I32], I32),
        "pnn_kernel_timing": ([V, I32, V, V], I32),
        "pnn_set_variant": ([V, I32], I32),
        "pnn_kernel_variant": ([V, P32], I32),
        "pnn_local_rows": ([V, I64, ctypes.POINTER(I64), ctypes.POINTER(I64)], I32),
        "pnn_merge_partial": ([V, V, V], I32),
        "pnn_merge_finish": ([V, V, V], I32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _ptr(t, dtype):
    import torch
    assert isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous() and t.dtype == dtype, \
        f"need a contiguous CUDA {dtype} tensor"
    return ctypes.c_void_p(t.data_ptr())


class PNN:
    """One handle of include/pnn.h.  Method names mirror the C entry points."""

    def __init__(self, layers, activation, init, n_subnets, lr, seed=0):
        self._L = load()
        layers = np.ascontiguousarray(layers, dtype=np.int32)
        act = np.ascontiguousarray([ACT[a] if isinstance(a, str) else a for a in activation], np.int32)
        init = INIT[init] if isinstance(init, str) else init
        h = ctypes.c_void_p()
        st = self._L.pnn_create(layers.ctypes.data_as(ctypes.c_void_p), len(layers),
                                act.ctypes.data_as(ctypes.c_void_p), int(init), int(n_subnets),
                                float(lr), int(seed) & (2**64 - 1), ctypes.byref(h))
        if st != PNN_OK:
            raise PnnError(st, self._L.pnn_last_error(None).decode())
        self.h = h
        self.layers = [int(v) for v in layers]
        self.n_subnets = int(n_subnets)

    # -- helpers ------------------------------------------------------------
    def _check(self, st):
        if st != PNN_OK:
            raise PnnError(st, self._L.pnn_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self._L.pnn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- ABI ------------------------------------------------------------------
    @property
    def param_count(self) -> int:
        return int(self._L.pnn_param_count(self.h))

    def set_comm(self, nranks, rank, unique_id: bytes | None = None):
        buf = None if unique_id is None else ctypes.create_string_buffer(bytes(unique_id), 128)
        self._check(self._L.pnn_set_comm(self.h, buf, int(nranks), int(rank)))

    def set_minibatch(self, batch, precision=PNN_FP32):
        self._check(self._L.pnn_set_minibatch(self.h, int(batch), int(precision)))

    def set_kernel(self, kernel):
        self._check(self._L.pnn_set_kernel(self.h, KERNEL[kernel] if isinstance(kernel, str) else kernel))

    def set_variant(self, variant):
        self._check(self._L.pnn_set_variant(self.h, VARIANT[variant] if isinstance(variant, str) else variant))

    def kernel_variant(self) -> int:
        v = ctypes.c_int32()
        self._check(self._L.pnn_kernel_variant(self.h, ctypes.byref(v)))
        return v.value

    def local_rows(self, n_total):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._L.pnn_local_rows(self.h, int(n_total), ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def merge_partial(self, sum_out, stream=None):
        import torch
        self._check(self._L.pnn_merge_partial(self.h, _ptr(sum_out, torch.float64), ctypes.c_void_p(_stream_ptr(stream))))

    def merge_finish(self, total, stream=None):
        import torch
        self._check(self._L.pnn_merge_finish(self.h, _ptr(total, torch.float64), ctypes.c_void_p(_stream_ptr(stream))))

    def train_epoch(self, x, labels, stream=None):
        import torch
        if x is None or x.shape[0] == 0:       # an idle rank (owns no CN): n = 0, NULL pointers
            self._check(self._L.pnn_train_epoch(self.h, None, None, 0, ctypes.c_void_p(_stream_ptr(stream))))
            return
        assert x.dim() == 2 and x.shape[1] == self.layers[0] and labels.shape == (x.shape[0],)
        self._check(self._L.pnn_train_epoch(self.h, _ptr(x, torch.float32), _ptr(labels, torch.int32),
                                            x.shape[0], ctypes.c_void_p(_stream_ptr(stream))))

    def train_epoch_host(self, x, labels, stream=None):
        """x, labels: host numpy arrays or CPU torch tensors (pinned preferred)."""
        import torch
        if isinstance(x, torch.Tensor):
            assert not x.is_cuda and x.is_contiguous() and x.dtype == torch.float32
            assert labels.is_contiguous() and labels.dtype == torch.int32
            xp, yp, n = x.data_ptr(), labels.data_ptr(), x.shape[0]
        else:
            x = np.ascontiguousarray(x, np.float32)
            labels = np.ascontiguousarray(labels, np.int32)
            xp, yp, n = x.ctypes.data, labels.ctypes.data, x.shape[0]
        self._check(self._L.pnn_train_epoch_host(self.h, ctypes.c_void_p(xp), ctypes.c_void_p(yp), n,
                                                 ctypes.c_void_p(_stream_ptr(stream))))

    def merge(self, stream=None):
        self._check(self._L.pnn_merge(self.h, ctypes.c_void_p(_stream_ptr(stream))))

    def predict(self, x, labels_out=None, subnet=-1, stream=None):
        import torch
        if labels_out is None:
            labels_out = torch.empty(x.shape[0], dtype=torch.int32, device=x.device)
        self._check(self._L.pnn_predict(self.h, int(subnet), _ptr(x, torch.float32), x.shape[0],
                                        _ptr(labels_out, torch.int32), ctypes.c_void_p(_stream_ptr(stream))))
        return labels_out

    def evaluate(self, x, labels, subnet=-1, stream=None):
        """(accuracy, confidence, cost) of the merged net (-1) or a local CN on
        labelled device rows (pnn_evaluate; fp64; synchronises the stream)."""
        import torch
        out = np.zeros(3, dtype=np.float64)
        self._check(self._L.pnn_evaluate(self.h, int(subnet), _ptr(x, torch.float32), _ptr(labels, torch.int32),
                                         x.shape[0], out.ctypes.data_as(ctypes.c_void_p),
                                         ctypes.c_void_p(_stream_ptr(stream))))
        return tuple(float(v) for v in out)

    def kernel_timing(self, enable):
        """Start (True) / stop (False) recording CUDA events around the training-kernel
        launches; stopping returns (mean ms per launch, launches)."""
        ms, n = ctypes.c_double(), ctypes.c_int32()
        self._check(self._L.pnn_kernel_timing(self.h, 1 if enable else 0, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def set_slots(self, slots):
        self._check(self._L.pnn_set_slots(self.h, int(slots)))

    def get_params(self, subnet=-1) -> np.ndarray:
        out = np.empty(self.param_count, dtype=np.float32)
        self._check(self._L.pnn_get_params(self.h, int(subnet), out.ctypes.data_as(ctypes.c_void_p), out.size))
        return out

    def set_params(self, params, subnet=-1):
        p = np.ascontiguousarray(params, dtype=np.float32)
        self._check(self._L.pnn_set_params(self.h, int(subnet), p.ctypes.data_as(ctypes.c_void_p), p.size))

    def device_params(self, subnet=-1) -> int:
        ptr = self._L.pnn_device_params(self.h, int(subnet))
        if not ptr:
            raise PnnError(PNN_ERR_INVALID, f"subnet {subnet} is not local")
        return ptr

    def local_subnets(self):
        a, b = ctypes.c_int32(), ctypes.c_int32()
        self._check(self._L.pnn_local_subnets(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def kernel_info(self):
        a, b = ctypes.c_int32(), ctypes.c_int32()
        self._check(self._L.pnn_kernel_info(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value
