"""Pins of the oracle's f2 evaluation metrics (SPEC.md's
cost/accuracy/confidence examples), CPU only:

* zero network, softmax output: every output is 1/10, so confidence = 0.1 and
  cost = ln 10 exactly (SPEC.md: "uniform 10-class output → ln(10)"); every
  logit ties, so the readout picks class 0 and accuracy = the share of label 0;
* zero network, sigmoid output: outputs 0.5 → confidence 0.5, cost ln 2;
* a "perfect" 10-10 softmax net (W = 1000·I on one-hot inputs): accuracy 1,
  confidence 1, cost 0 (exp(−1000) underflows to 0 in fp64);
* random softmax nets: cost = mean of the oracle's per-sample Eq.6 cost
  (orc_cost, an independent C path), confidence ∈ [1/10, 1].
"""
import math

import numpy as np

from datagen import make_split


def test_uniform_softmax_net(orc):
    layers = [784, 16, 10]
    P = orc.param_count(layers)
    X, y = make_split(300, "test", 0)
    acc, conf, cost = orc.evaluate(layers, ["relu", "softmax"], np.zeros(P), X, y)
    assert abs(conf - 0.1) < 1e-15
    assert abs(cost - math.log(10)) < 1e-12
    assert acc == np.mean(y == 0)


def test_uniform_sigmoid_net(orc):
    layers = [784, 8, 10]
    P = orc.param_count(layers)
    X, y = make_split(50, "test", 0)
    acc, conf, cost = orc.evaluate(layers, ["sigmoid", "sigmoid"], np.zeros(P), X, y)
    assert conf == 0.5 and abs(cost - math.log(2)) < 1e-15


def test_perfect_net():
    import oracle as orc
    y = np.arange(40, dtype=np.int32) % 10
    X = np.eye(10)[y]
    p = np.concatenate([(1000.0 * np.eye(10)).ravel(), np.zeros(10)])
    acc, conf, cost = orc.evaluate([10, 10], ["softmax"], p, X, y)
    assert (acc, conf, cost) == (1.0, 1.0, 0.0)


def test_cost_matches_per_sample_eq6(orc):
    rng = np.random.default_rng(3)
    layers, act = [20, 12, 10], ["tanh", "softmax"]
    P = orc.param_count(layers)
    p = rng.normal(scale=0.8, size=P)
    X = rng.random((60, 20))
    y = rng.integers(0, 10, 60).astype(np.int32)
    acc, conf, cost = orc.evaluate(layers, act, p, X, y)
    per = [orc.cost(layers, act, p, X[i], int(y[i])) for i in range(60)]
    assert abs(cost - np.mean(per)) < 1e-12
    assert 0.1 <= conf <= 1.0
    assert acc == np.mean(orc.predict(layers, act, p, X) == y)
