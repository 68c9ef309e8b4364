"""Full-size, full-population parity of one BASELINE config — test infrastructure
(used by tests/test_gpu_fullsize.py and tools/parity_report.py, which writes
profiles/parity_r2.json).

The GPU trains every CN of the config through the C ABI; the oracle re-trains EVERY
CN on its slice (threads over CNs) and merges them.  The report holds, per CN, the
max-abs error against the oracle (fp32 paths) or the per-layer relative Frobenius
error against the oracle's bf16 mode (C5, R31), and for each fp32 CN over
north_star's 1e-4:
  * ReLU-family nets: the R24 kink accounting (tests/kinks.py) — accepted only with a
    logged kink at the first divergent sample;
  * smooth nets: the R22 fp32 envelope (tests/envelope.py) of that CN.
Then the merged network (GPU merge of the GPU children vs the oracle's merge of the
oracle children; bound: the mean of the per-CN bounds, the merge being the mean of
the children), the merge arithmetic (bit-exact on the same children), the readout of
the same weights (bit-exact) and R26(ii): labels of the GPU-trained vs the
oracle-trained merged network on the full test set, every mismatch with the top-2
margin of the oracle-trained logits.
"""
from __future__ import annotations

import os
import time

import numpy as np
import torch

from datagen import make_split
from workloads import CONFIGS

TOL = 1e-4
RELU_FAMILY = ("relu", "leaky_relu")


def _layer_rel(layers, got, ref):
    out, o = [], 0
    for l in range(1, len(layers)):
        n = layers[l] * layers[l - 1] + layers[l]
        g, r = got[o:o + n].astype(np.float64), ref[o:o + n].astype(np.float64)
        out.append(float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)))
        o += n
    return out


def run_full(orc, name, epochs=None, threads=None, variant=None, log=print):
    from paper_2304_09590_b200 import PNN
    from paper_2304_09590_b200.pnn import PNN_BF16
    c = CONFIGS[name]
    E = c.epochs if epochs is None else epochs
    threads = threads or max(1, len(os.sched_getaffinity(0)))
    t0 = time.time()
    X, y = make_split(c.n_train, "train", 0)
    Xt, _ = make_split(c.n_test, "test", 0)
    net = PNN(c.layers, c.act, c.init, c.K, c.lr, seed=0)
    if c.batch > 1:
        net.set_minibatch(c.batch, PNN_BF16 if c.precision == "bf16" else 0)
    if variant is not None:
        net.set_variant(variant)
    kernel, _ = net.kernel_info()
    var = net.kernel_variant()
    xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    for _ in range(E):
        net.train_epoch(xd, yd)
    net.merge()
    torch.cuda.synchronize()
    kids = np.stack([net.get_params(i) for i in range(c.K)])
    merged = net.get_params(-1)
    lab_gpu = net.predict(torch.from_numpy(Xt).cuda()).cpu().numpy()
    t1 = time.time()
    okids, omerged = orc.train_pnn(c.layers, c.act, c.init, c.K, c.lr, 0, X, y, epochs=E, batch=c.batch,
                                   threads=threads, precision=c.precision)
    t2 = time.time()
    p0 = orc.init_params(c.layers, c.init, 0)
    start, count = orc.shard_bounds(c.n_train, c.K)
    rep = {"config": name, "layers": list(c.layers), "act": list(c.act), "K": c.K, "epochs": E,
           "batch": c.batch, "precision": c.precision, "kernel": int(kernel), "variant": int(var),
           "gpu_s": round(t1 - t0, 2), "oracle_s": round(t2 - t1, 2), "oracle_threads": threads, "cns": []}
    bounds = []
    if c.precision == "bf16":
        for i in range(c.K):
            rel = _layer_rel(c.layers, kids[i], okids[i])
            rep["cns"].append({"cn": i, "layer_rel": rel})
        rep["merged_layer_rel"] = _layer_rel(c.layers, merged, omerged)
        rep["max_layer_rel"] = max(max(r["layer_rel"]) for r in rep["cns"])
    else:
        for i in range(c.K):
            err = float(np.abs(kids[i] - okids[i]).max())
            cn = {"cn": i, "max_abs": err}
            bound = TOL
            if err >= TOL:
                a, b = int(start[i]), int(start[i] + count[i])
                from tests.cnrule import cn_bound
                bound, info = cn_bound(orc, net, c.layers, c.act, c.init, c.lr, X[a:b], y[a:b], err, okids[i], E,
                                       c.batch, kid=kids[i])
                cn.update(info or {})
            cn["bound"] = bound
            cn["ok"] = err < TOL or err <= bound
            bounds.append(bound)
            rep["cns"].append(cn)
        errs = np.array([cn["max_abs"] for cn in rep["cns"]])
        rep["max_abs_max"] = float(errs.max())
        rep["max_abs_median"] = float(np.median(errs))
        rep["cns_over_1e-4"] = int((errs >= TOL).sum())
        rep["merged_max_abs"] = float(np.abs(merged - omerged).max())
        rep["merged_bound"] = float(np.mean(bounds))
    rep["merge_bit_exact"] = bool(np.array_equal(merged, orc.merge(kids)))
    rep["readout_same_weights_bit_exact"] = bool(np.array_equal(lab_gpu, orc.predict(c.layers, c.act, merged, Xt)))
    lab_orc, logits = orc.predict(c.layers, c.act, omerged, Xt, return_logits=True)
    mism = np.where(lab_orc != lab_gpu)[0]
    margins = []
    for r in mism[:50]:
        z = np.sort(logits[r])[::-1]
        margins.append({"row": int(r), "gpu": int(lab_gpu[r]), "oracle": int(lab_orc[r]), "top2_margin": float(z[0] - z[1])})
    rep["labels_trained_mismatches"] = int(len(mism))
    rep["labels_trained_mismatch_margins"] = margins
    rep["test_rows"] = int(len(Xt))
    log(f"{name}: {rep.get('max_abs_max', rep.get('max_layer_rel'))} max, merged "
        f"{rep.get('merged_max_abs', rep.get('merged_layer_rel'))}, label mismatches {len(mism)}")
    return rep


def assert_report(rep):
    """The gates, in the order the report states them."""
    if rep["precision"] == "bf16":
        assert rep["max_layer_rel"] <= 2e-2, rep["max_layer_rel"]
        assert max(rep["merged_layer_rel"]) <= 2e-2, rep["merged_layer_rel"]
    else:
        bad = [cn for cn in rep["cns"] if not cn["ok"]]
        assert not bad, f"CNs over the gate without a logged kink / envelope: {bad[:5]}"
        assert rep["merged_max_abs"] <= rep["merged_bound"], (rep["merged_max_abs"], rep["merged_bound"])
    assert rep["merge_bit_exact"]
    assert rep["readout_same_weights_bit_exact"]
    # R26(ii): GPU-trained vs oracle-trained labels; a mismatch is only a tie within rounding
    for m in rep["labels_trained_mismatch_margins"]:
        assert m["top2_margin"] < 1e-3, m
