#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g_pytest.log
for c in C4 F1; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value']/1e6, d['roofline']['frac'], d['roofline']['train_ms_per_launch'], d['breakdown_ms'])"; done
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/g_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_resident -s 3 -c 1 -o gpurun_out/prof_resident_C4 $B > gpurun_out/g_ncu.log 2>&1; echo "ncu rc=$?"
