#!/bin/bash
cd /root/repo 2>/dev/null || cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "reduced or c4_full or c1_full or leaky or determinism or host_input or slots or c2_full" 2>&1 | tail -3
for v in "" _v8; do
  echo "== '$v'"
  PNN_LIB=$PWD/paper_2304_09590_b200/libpnn$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value']/1e6, d['roofline']['frac'], d['roofline']['train_ms_per_launch'], d['clocks']['sm_mhz'])"
done
timeout 120 python tools/trace_resident.py --config C4 --K 148 --rows 256 2>&1 | grep -A1 "cta 0 warp" | head -8
