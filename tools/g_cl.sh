#!/bin/bash
cd /root/repo 2>/dev/null || cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster or reduced" 2>&1 | tail -5
for c in C3 C2 C4; do timeout 600 python bench.py --config $c --kernel cluster --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value']/1e6, d['config']['kernel'], d['roofline']['frac'], d['roofline']['train_ms_per_launch'], d['ms_per_step'])"; done
