"""CPU checks of two readings the GPU path relies on, fp32 arithmetic
emulated with numpy:

* R32: the deep variant's chain forms tanh(z) = 1 - 2/(1 + e^{2z}) and
  sigmoid(z) = 1/(1 + e^{-z}); in fp32 both stay within ~1e-7 absolute of the exact
  functions over the range activations take (the GPU adds ex2.approx / rcp.approx
  rounding of the same order);
* R27: W(t)·x = W(t-L)·x - Σ_k g(t-k) (x(t-k)·x),
  the identity the resident kernels' lookahead uses, holds to fp32 rounding.
"""
import numpy as np


def test_r32_tanh_sigmoid_forms():
    z = np.linspace(-30, 30, 200001).astype(np.float32)
    f32 = np.float32
    t = f32(1) - f32(2) / (f32(1) + np.exp(f32(2) * z, dtype=np.float32))
    s = f32(1) / (f32(1) + np.exp(-z, dtype=np.float32))
    zd = z.astype(np.float64)
    assert np.abs(t.astype(np.float64) - np.tanh(zd)).max() < 2.5e-7
    assert np.abs(s.astype(np.float64) - 1.0 / (1.0 + np.exp(-zd))).max() < 1.5e-7


def test_r27_lookahead_identity():
    rng = np.random.default_rng(3)
    D, H, L = 784, 64, 4
    W0 = rng.normal(size=(H, D)).astype(np.float64)
    xs = rng.random((L + 1, D))
    g = rng.normal(scale=1e-3, size=(L, H))
    W = W0.copy()
    for k in range(L):                 # eager: W -= g(k) x(k)ᵀ, then the forward of x(L)
        W -= np.outer(g[k], xs[k])
    eager = W @ xs[L]
    lazy = W0 @ xs[L] - sum(g[k] * (xs[k] @ xs[L]) for k in range(L))
    np.testing.assert_allclose(lazy, eager, rtol=0, atol=1e-10)
