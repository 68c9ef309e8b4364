"""The per-CN parity rule of the fp32 paths — test infrastructure (DESIGN.md §3 R22/R24).

north_star: every weight and bias of every CN and of the merged net within max-abs 1e-4
of the fp32 oracle.  A CN over that bar passes only with a recorded cause:
  * ReLU-family hidden layers (Eq.4's branch point): a logged kink at
    the first divergent step (R24, tests/kinks.py) — a pre-activation within 1e-5 of 0
    whose sign the two sides' rounding decides differently;
  * otherwise (smooth hidden layers, or a ReLU CN whose divergence grows gradually with
    no kink — N(0,1)-init nets at η = 0.1 are as ill-conditioned in fp32 as C2): the
    CN's error is inside the fp32 envelope of its slice
    (R22, tests/envelope.py): no larger than the oracle's own spread under 1-ulp
    perturbations of its inputs (64 trials: a further valid trajectory lands outside with
    probability ~1/65) or the spread of another valid fp32
    ordering (torch: BLAS summation order, per-sample or mini-batch);
  * beyond the envelope (R34): the GPU is no farther from the same algorithm run in fp64
    than the fp32 oracle is — when fp32 cannot fix the trajectory to 1e-4, the GPU must be
    at least as accurate as the oracle it is compared with.
The merged net is the mean of the children, so its bound is the mean of their bounds.
"""
from __future__ import annotations

import numpy as np

TOL = 1e-4
RELU_FAMILY = ("relu", "leaky_relu")


def _kernel_name(kid):
    return {1: "reference", 2: "resident", 5: "cluster"}.get(int(kid), "auto")


def cn_bound(orc, net, layers, act, init, lr, Xi, yi, err, okid, epochs, batch=1, kid=None):
    """(bound, info) for one CN whose max-abs error is `err` (`kid`: the GPU's parameters,
    for the R34 accuracy check)."""
    if err < TOL:
        return TOL, None
    p0 = orc.init_params(layers, init, 0)
    info = {}
    if any(a in RELU_FAMILY for a in act[:-1]):
        from tests.kinks import find_kink, has_kink
        kr = find_kink(orc, list(layers), list(act), lr, p0, Xi, yi, epochs, variant=net.kernel_variant(),
                       kernel=_kernel_name(net.kernel_info()[0]), batch=batch)
        info = {"kink": kr, "kink_logged": has_kink(kr)}
        if has_kink(kr):
            return err, info
        # no kink: a gradual divergence — the slice is ill-conditioned in fp32 (R22, as C2)
    from tests.envelope import perturbation_envelope, torch_sgd_fp32
    env = perturbation_envelope(orc, layers, act, p0, Xi, yi, lr, epochs, batch=batch)
    if all(a in ("sigmoid", "tanh", "relu", "softmax") for a in act):
        env = max(env, float(np.abs(torch_sgd_fp32(layers, act, p0, Xi, yi, lr, epochs, batch) - okid).max()))
    info["envelope"] = env
    bound = max(TOL, env)
    if err > bound and kid is not None:
        # R34: fp32 does not fix this trajectory to 1e-4; judge both fp32 realisations by the
        # same algorithm in fp64 (the oracle's exact-arithmetic stand-in): the GPU passes if it
        # is no farther from that than the fp32 oracle itself is.
        o64 = orc.train(layers, act, p0.astype(np.float64), np.asarray(Xi, np.float64), yi, lr, epochs,
                        batch=batch, dtype=np.float64)
        d_gpu = float(np.abs(np.asarray(kid, np.float64) - o64).max())
        d_orc = float(np.abs(np.asarray(okid, np.float64) - o64).max())
        info["fp64"] = {"gpu_vs_fp64": d_gpu, "oracle32_vs_fp64": d_orc}
        if d_gpu <= d_orc:
            bound = err
    return bound, info


def check_cns(orc, net, layers, act, init, K, lr, X, y, kids, okids, epochs, batch=1, log=print):
    start, count = orc.shard_bounds(len(y), K)
    bounds, report = [], []
    for i in range(K):
        err = float(np.abs(kids[i] - okids[i]).max())
        a, b = int(start[i]), int(start[i] + count[i])
        bound, info = cn_bound(orc, net, layers, act, init, lr, X[a:b], y[a:b], err, okids[i], epochs, batch,
                               kid=kids[i])
        report.append((i, err, bound, info))
        bounds.append(bound)
        assert err < TOL or err <= bound, f"CN {i}: max-abs {err:.3g} without a recorded cause: {info}"
    log("per-CN (index, max-abs, bound, cause):", report)
    return bounds


def check_merged(merged, omerged, bounds):
    err = float(np.abs(merged - omerged).max())
    assert err <= float(np.mean(bounds)), f"merged max-abs {err:.3g} > mean of the per-CN bounds {np.mean(bounds):.3g}"
