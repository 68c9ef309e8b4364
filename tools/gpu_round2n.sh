#!/bin/bash
# Round-2 batch (n): Gram pre-pass chunking / ring-depth A/B, parity on the new chunking. The gfix / gs4 / gs8 libraries were
# experiment-only builds (-DPNN_GRAM_FIXED_CHUNK, -DPNN_GRAM_SLOTS=4|8); those switches were removed after the A/B
# (results: profiles/README.md, r2r), so this script documents the run and no longer reproduces it.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/r2n; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
for v in main gfix gs4 gs8; do
  L=$PWD/paper_2304_09590_b200/libpnn_$v.so; [ $v = main ] && L=$PWD/paper_2304_09590_b200/libpnn.so
  PNN_LIB=$L timeout 300 $B > $O/bench_${v}_$rep.json 2> $O/bench_${v}_$rep.err; echo "bench $v rc=$?"
  python - <<PY
import json
d=json.loads(open("$O/bench_${v}_$rep.json").read().strip().splitlines()[-1]); r=d["roofline"]
print("$v", round(d["value"]/1e6,2), "ms/step", round(d["ms_per_step"],3), "sgd", round(r["kernel_ms_per_launch"],3), "train", round(r["train_ms_per_epoch"],3), "gram", round(r["train_ms_per_epoch"]-r["kernel_ms_per_launch"],3))
PY
done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deep.py tests/test_gpu_fullsize.py -q -k "not c5 and not C5" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
