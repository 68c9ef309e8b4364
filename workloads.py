"""BASELINE.json configs C1-C5 as data (shapes, activations, init, K, η, epochs).

Shared by tests and bench.py.  No method arithmetic.
"""
from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    layers: tuple
    act: tuple
    init: str
    K: int
    lr: float
    n_train: int
    n_test: int
    epochs: int = 1
    batch: int = 1
    precision: str = "fp32"
    note: str = ""


CONFIGS = {
    # configs[0]: 784-16-10 sigmoid/sigmoid, U[-.5,.5], K=1, SGD η=0.1, MSE (R11), 1000/200
    "C1": Config("C1", (784, 16, 10), ("sigmoid", "sigmoid"), "uniform", 1, 0.1, 1000, 200),
    # configs[1]: 784-100-10 sigmoid (R12: sigmoid output + ½-SSE), K=4, η=0.1, 60k/10k;
    # init unstated → the paper's own N(0,1)
    "C2": Config("C2", (784, 100, 10), ("sigmoid", "sigmoid"), "normal", 4, 0.1, 60000, 10000),
    # configs[2]: 784-300-100-10 tanh/softmax+CE, Xavier-normal, K=32, η=0.01, 5 epochs
    "C3": Config("C3", (784, 300, 100, 10), ("tanh", "tanh", "softmax"), "xavier", 32, 0.01,
                 60000, 10000, epochs=5),
    # configs[3]: 784-128-10 ReLU/softmax, He-normal, K=1024 (128/GPU × 8), η=0.01, 2^20 rows
    "C4": Config("C4", (784, 128, 10), ("relu", "softmax"), "he", 1024, 0.01, 1 << 20, 10000),
    # configs[4]: 784-1024-1024-10 ReLU (R13: softmax+CE output), K=8, mini-batch 64, η=0.05,
    # 480k rows, 3 epochs; bf16 operands / fp32 accumulate + master (R25) on tcgen05 (a10)
    "C5": Config("C5", (784, 1024, 1024, 10), ("relu", "relu", "softmax"), "he", 8, 0.05,
                 480000, 10000, epochs=3, batch=64, precision="bf16",
                 note="init unstated; He-normal (ReLU)"),
    # §8(f) f1: the paper's own workload: 784-256-10 ReLU +
    # softmax/CE, N(0,1) init (the paper's NormFloat64, :209-213), fp32 mini-batch B=50,
    # η 0.1 (Fig.3; Fig.2 uses 0.05), K=10 CNs, 20 epochs, 60k/10k rows
    "F1": Config("F1", (784, 256, 10), ("relu", "softmax"), "normal", 10, 0.1, 60000, 10000,
                 epochs=20, batch=50, note="paper's Fig.3 setting"),
}
