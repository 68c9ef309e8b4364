"""CPU oracle of the PNN hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The product package
(paper_2304_09590_b200) never imports it and shares no code with it.

The arithmetic lives in oracle/oracle.c (+ oracle_body.h), plain C built with
``gcc -O2 -ffp-contract=off``; this module only marshals numpy arrays and
composes the per-network calls into the paper's PNN procedure
(PAPER.md:166-172, 225-238):

  1. init one network and clone it K times          (R16)
  2. split the data into K contiguous slices        (R17)
  3. train every child on its slice independently
  4. average all weights and biases

Nothing here is "parity unpinned": each function is pinned by
tests/test_oracle_*.py (closed forms, finite differences, a torch-fp64
library pin, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

SIGMOID, TANH, RELU, SOFTMAX, LEAKY_RELU = 0, 1, 2, 3, 4
INIT_NORMAL, INIT_UNIFORM, INIT_XAVIER, INIT_HE = 0, 1, 2, 3
ACT_NAMES = {"sigmoid": SIGMOID, "tanh": TANH, "relu": RELU, "softmax": SOFTMAX, "leaky_relu": LEAKY_RELU}
INIT_NAMES = {"normal": INIT_NORMAL, "uniform": INIT_UNIFORM, "xavier": INIT_XAVIER, "he": INIT_HE}

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2 -ffp-contract=off, no fast-math)."""
    src = [os.path.join(HERE, "oracle.c")]
    deps = src + [os.path.join(HERE, "oracle_body.h")]
    if (not force and os.path.exists(LIB_PATH)
            and all(os.path.getmtime(LIB_PATH) >= os.path.getmtime(d) for d in deps)):
        return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                           "-fPIC", "-shared", "-o", tmp] + src + ["-lm"])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P, I, I64, D, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_float
        for suf, R in (("_f32", F), ("_f64", D)):
            getattr(L, "orc_forward" + suf).argtypes = [P, I, P, P, P, P, P]
            getattr(L, "orc_forward" + suf).restype = None
            getattr(L, "orc_cost" + suf).argtypes = [P, I, P, P, P, I, P]
            getattr(L, "orc_cost" + suf).restype = D
            getattr(L, "orc_train" + suf).argtypes = [P, I, P, P, P, P, ctypes.c_long, R, I, I]
            getattr(L, "orc_train" + suf).restype = I
            getattr(L, "orc_predict" + suf).argtypes = [P, I, P, P, P, ctypes.c_long, P, P]
            getattr(L, "orc_predict" + suf).restype = I
        L.orc_uniform.argtypes = [ctypes.c_uint64, I, I, I64, I]
        L.orc_uniform.restype = D
        L.orc_normal.argtypes = [ctypes.c_uint64, I, I, I64]
        L.orc_normal.restype = D
        L.orc_init.argtypes = [P, I, I, ctypes.c_uint64, P]
        L.orc_init.restype = I
        L.orc_param_count.argtypes = [P, I]
        L.orc_bf16_round.argtypes = [ctypes.c_float]
        L.orc_bf16_round.restype = ctypes.c_float
        L.orc_train_bf16.argtypes = [P, I, P, P, P, P, ctypes.c_long, ctypes.c_float, I, I]
        L.orc_train_bf16.restype = I
        L.orc_param_count.restype = ctypes.c_long
        L.orc_shard_bounds.argtypes = [ctypes.c_long, I, P, P]
        L.orc_shard_bounds.restype = None
        L.orc_merge.argtypes = [P, I, ctypes.c_long, P]
        L.orc_merge.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _net(layers, act):
    layers = np.ascontiguousarray(layers, dtype=np.int32)
    act = np.ascontiguousarray([ACT_NAMES[a] if isinstance(a, str) else a for a in act],
                               dtype=np.int32)
    assert len(act) == len(layers) - 1
    return layers, act, len(layers) - 1


def _dt(dtype):
    dtype = np.dtype(dtype)
    assert dtype in (np.float32, np.float64)
    return dtype, ("_f32" if dtype == np.float32 else "_f64")


def param_count(layers) -> int:
    layers = np.ascontiguousarray(layers, dtype=np.int32)
    return int(lib().orc_param_count(_p(layers), len(layers) - 1))


def layer_views(params: np.ndarray, layers):
    """[(W^l [n_l, n_{l-1}], b^l [n_l]) for l = 1..L] views into a flat vector."""
    out, off = [], 0
    for l in range(1, len(layers)):
        nin, nout = int(layers[l - 1]), int(layers[l])
        W = params[off:off + nin * nout].reshape(nout, nin)
        off += nin * nout
        b = params[off:off + nout]
        off += nout
        out.append((W, b))
    return out


def init_params(layers, init, seed: int) -> np.ndarray:
    layers = np.ascontiguousarray(layers, dtype=np.int32)
    init = INIT_NAMES[init] if isinstance(init, str) else init
    out = np.empty(param_count(layers), dtype=np.float32)
    rc = lib().orc_init(_p(layers), len(layers) - 1, int(init), seed & (2**64 - 1), _p(out))
    if rc != 0:
        raise ValueError(f"unknown init {init}")
    return out


def uniform(seed, layer, kind, index, s=0) -> float:
    return lib().orc_uniform(seed, layer, kind, index, s)


def normal(seed, layer, kind, index) -> float:
    return lib().orc_normal(seed, layer, kind, index)


def forward(layers, act, params, x0, dtype=np.float64):
    """One sample: returns (z list, x list) per layer l = 1..L (Eqs.2-5)."""
    layers, act, L = _net(layers, act)
    dtype, suf = _dt(dtype)
    params = np.ascontiguousarray(params, dtype=dtype)
    x0 = np.ascontiguousarray(x0, dtype=dtype)
    tot = int(layers[1:].sum())
    zs = np.empty(tot, dtype=dtype)
    xs = np.empty(tot, dtype=dtype)
    getattr(lib(), "orc_forward" + suf)(_p(layers), L, _p(act), _p(params), _p(x0), _p(zs), _p(xs))
    zl, xl, off = [], [], 0
    for l in range(1, L + 1):
        zl.append(zs[off:off + layers[l]].copy())
        xl.append(xs[off:off + layers[l]].copy())
        off += layers[l]
    return zl, xl


def cost(layers, act, params, x0, label, dtype=np.float64) -> float:
    layers, act, L = _net(layers, act)
    dtype, suf = _dt(dtype)
    params = np.ascontiguousarray(params, dtype=dtype)
    x0 = np.ascontiguousarray(x0, dtype=dtype)
    scratch = np.empty(2 * int(layers[1:].sum()), dtype=dtype)
    return getattr(lib(), "orc_cost" + suf)(_p(layers), L, _p(act), _p(params), _p(x0),
                                           int(label), _p(scratch))


def bf16_round(v: float) -> float:
    """bfloat16 round-to-nearest-even of one fp32 value (reading R25)."""
    return float(lib().orc_bf16_round(float(v)))


def train(layers, act, params, X, y, lr, epochs=1, batch=1, dtype=np.float32,
          precision="fp32") -> np.ndarray:
    """Train ONE network over rows X in order; returns the new parameters.
    precision="bf16": the mini-batch variant with R25's bf16 rounding points
    (fp32 master weights, fp32 accumulation); always fp32 arithmetic."""
    layers, act, L = _net(layers, act)
    if precision == "bf16":
        out = np.array(params, dtype=np.float32, copy=True)
        X = np.ascontiguousarray(X, dtype=np.float32)
        y = np.ascontiguousarray(y, dtype=np.int32)
        assert X.shape == (len(y), layers[0])
        rc = lib().orc_train_bf16(_p(layers), L, _p(act), _p(out), _p(X), _p(y), len(y), float(lr),
                                  int(epochs), int(batch))
        if rc != 0:
            raise MemoryError("oracle allocation failed")
        return out
    dtype, suf = _dt(dtype)
    out = np.array(params, dtype=dtype, copy=True)
    X = np.ascontiguousarray(X, dtype=dtype)
    y = np.ascontiguousarray(y, dtype=np.int32)
    assert X.shape == (len(y), layers[0])
    rc = getattr(lib(), "orc_train" + suf)(_p(layers), L, _p(act), _p(out), _p(X), _p(y),
                                          len(y), float(lr), int(epochs), int(batch))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return out


def predict(layers, act, params, X, dtype=np.float64, return_logits=False):
    """Labels = argmax of z^L, ties to the lowest index (R19)."""
    layers, act, L = _net(layers, act)
    dtype, suf = _dt(dtype)
    params = np.ascontiguousarray(params, dtype=dtype)
    X = np.ascontiguousarray(X, dtype=dtype)
    n = X.shape[0]
    labels = np.empty(n, dtype=np.int32)
    logits = np.empty((n, layers[-1]), dtype=dtype) if return_logits else None
    getattr(lib(), "orc_predict" + suf)(_p(layers), L, _p(act), _p(params), _p(X), n,
                                       _p(labels), _p(logits) if logits is not None else None)
    return (labels, logits) if return_logits else labels


def evaluate(layers, act, params, X, y):
    """f2 evaluation metrics of one network on labelled rows, in fp64:

    * accuracy   = fraction of rows whose readout label (predict, R19) equals y;
    * confidence = mean over rows of max_k x^L_k, x^L the output activation (softmax:
      the predicted class's probability; undefined in the paper, reading R29);
    * cost       = mean over rows of −log(max(x^L_y, 1e-12)) (Eq.6, PAPER.md:100-103:
      C = −Σ_i e_i log x_i with one-hot e; ε-clamp R29).
    x^L from the fp64 logits z^L: softmax exp(z − max z)/Σ (Eq.5 with R4), else φ_L(z)
    (sigmoid 1/(1+e^−z), tanh, ReLU, leaky ReLU (R30) as in Eqs.3-4)."""
    layers_, act_, L = _net(layers, act)
    labels, z = predict(layers, act, params, X, return_logits=True)
    a = int(act_[-1])
    if a == SOFTMAX:
        e = np.exp(z - z.max(axis=1, keepdims=True))
        x = e / e.sum(axis=1, keepdims=True)
    elif a == SIGMOID:
        x = 1.0 / (1.0 + np.exp(-z))
    elif a == TANH:
        x = np.tanh(z)
    elif a == RELU:
        x = np.where(z >= 0, z, 0.0)
    else:
        x = np.where(z >= 0, z, float(np.float32(0.01)) * z)
    y = np.asarray(y, dtype=np.int64)
    rows = np.arange(len(y))
    acc = float(np.mean(labels == y))
    conf = float(np.mean(x.max(axis=1)))
    cost = float(np.mean(-np.log(np.maximum(x[rows, y], 1e-12))))
    return acc, conf, cost


def shard_bounds(N: int, K: int):
    start = np.empty(K, dtype=np.int64)
    count = np.empty(K, dtype=np.int64)
    lib().orc_shard_bounds(N, K, _p(start), _p(count))
    return start, count


def merge(children: np.ndarray) -> np.ndarray:
    children = np.ascontiguousarray(children, dtype=np.float32)
    K, P = children.shape
    out = np.empty(P, dtype=np.float32)
    lib().orc_merge(_p(children), K, P, _p(out))
    return out


def train_pnn(layers, act, init, K, lr, seed, X, y, epochs=1, batch=1, dtype=np.float32,
              threads=1, subnets=None, init_params_=None, precision="fp32"):
    """The paper's PNN procedure.  Returns (children [K or len(subnets), P], merged or None).

    ``subnets`` restricts training to those child indices (full-size sampled
    parity); the merge is only computed when every child is trained.
    ``X``/``y`` may be a callable (start, count) -> (X, y) so that a sampled
    run only materialises the rows it needs.
    """
    p0 = init_params(layers, init, seed) if init_params_ is None else np.asarray(init_params_, np.float32)
    N = len(y) if not callable(X) else None
    if N is None:
        raise ValueError("pass N via X arrays, or use train_pnn_rows")
    return _train_children(layers, act, p0, K, lr, N, lambda s, c: (X[s:s + c], y[s:s + c]),
                           epochs, batch, dtype, threads, subnets, precision)


def train_pnn_rows(layers, act, init, K, lr, seed, N, rows, epochs=1, batch=1,
                   dtype=np.float32, threads=1, subnets=None, precision="fp32"):
    p0 = init_params(layers, init, seed)
    return _train_children(layers, act, p0, K, lr, N, rows, epochs, batch, dtype, threads, subnets,
                           precision)


def _train_children(layers, act, p0, K, lr, N, rows, epochs, batch, dtype, threads, subnets,
                    precision="fp32"):
    start, count = shard_bounds(N, K)
    idx = list(range(K)) if subnets is None else list(subnets)

    def one(i):
        Xi, yi = rows(int(start[i]), int(count[i]))
        return train(layers, act, p0, Xi, yi, lr, epochs, batch, dtype, precision).astype(np.float32)

    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            kids = list(ex.map(one, idx))
    else:
        kids = [one(i) for i in idx]
    children = np.stack(kids)
    merged = merge(children) if subnets is None else None
    return children, merged
