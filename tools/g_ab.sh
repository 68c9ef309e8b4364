#!/bin/bash
cd /root/repo 2>/dev/null || cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "reduced or c4_full or short_slices or leaky or determinism" 2>&1 | tail -2
for v in "" _base "" _base; do
  echo "== '$v'"
  PNN_LIB=$PWD/paper_2304_09590_b200/libpnn$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value']/1e6, d['roofline']['frac'], d['roofline']['train_ms_per_launch'], d['clocks']['sm_mhz'])"
done
