#!/bin/bash
# Round-2 batch (o): Gram pre-pass with contiguous per-warp chunks + compile-time ring slots: parity, bench, ncu of the pre-pass.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-r2o}; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do timeout 300 $B > $O/bench_$rep.json 2> $O/bench_$rep.err; echo "bench rc=$?"
python - <<PY
import json
d=json.loads(open("$O/bench_$rep.json").read().strip().splitlines()[-1]); r=d["roofline"]
print(round(d["value"]/1e6,2), "ms/step", round(d["ms_per_step"],3), "sgd", round(r["kernel_ms_per_launch"],3), "train", round(r["train_ms_per_epoch"],3), "gram", round(r["train_ms_per_epoch"]-r["kernel_ms_per_launch"],3))
PY
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deep.py tests/test_gpu_fullsize.py -q -k "not c5 and not C5" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
B1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram -s 3 -c 1 -o $O/prof_gram_C4 $B1 > $O/ncu_gram.log 2>&1; echo "ncu gram rc=$?"
