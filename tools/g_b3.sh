#!/bin/bash
cd /root/repo 2>/dev/null || cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_minibatch_bf16.py -q -x 2>&1 | tail -3
python tools/c5_small.py 64
timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['value']/1e6, d['roofline'])"
