#!/bin/bash
cd /root/repo 2>/dev/null || cd "$(dirname "$0")/.."
for c in C1 C2 C3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value']/1e6, d['config']['kernel'], d['roofline']['frac'], d['roofline']['train_ms_per_launch'], d['ms_per_step'])"; done
