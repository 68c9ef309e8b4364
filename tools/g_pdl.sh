#!/bin/bash
cd /root/repo 2>/dev/null || cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_minibatch_bf16.py tests/test_gpu_tcgemm.py tests/test_gpu_parity.py -q -x -k "minibatch or f1 or tc_gemm or bf16 or evaluate" 2>&1 | tail -3
python tools/c5_small.py 64
for c in C5 F1 C4; do timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value']/1e6, d['roofline']['frac'], d['roofline']['train_ms_per_launch'], d['breakdown_ms'])"; done
