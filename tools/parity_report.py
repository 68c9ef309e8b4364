"""Full-size, full-population parity report of the BASELINE configs -> JSON (tools only).

    python tools/parity_report.py [--configs C1,C2,C3,C4,C5] [--out profiles/parity_r2.json]

C5 runs one epoch (its oracle bf16 mode costs ~6 min of the box's cores per epoch).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from tests.fullsize import run_full  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
ap.add_argument("--out", default="gpurun_out/parity_r2.json")
a = ap.parse_args()
oracle.build()
out = {}
for name in a.configs.split(","):
    rep = run_full(oracle, name, epochs=1 if name == "C5" else None)
    if name in ("C4",):                        # 1024 CNs: keep the per-CN list compact
        rep["cns"] = [cn for cn in rep["cns"] if cn["max_abs"] >= 1e-5] + \
            [{"summary": "CNs with max-abs < 1e-5 omitted", "count": sum(1 for cn in rep["cns"] if cn["max_abs"] < 1e-5)}]
    out[name] = rep
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1, default=float)
print(json.dumps({k: {kk: v[kk] for kk in v if kk not in ("cns",)} for k, v in out.items()}, default=float)[:4000])
