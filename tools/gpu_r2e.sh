#!/bin/bash
# round 2e: first GPU run of the warp-specialised TMEM variant (v12, k_ws.cu)
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ws" > gpurun_out/r2e_pytest_ws.log 2>&1
echo "pytest ws exit $?" >> gpurun_out/r2e_pytest_ws.log
for v in ws tmem v8; do
  timeout 300 python bench.py --steps 5 --warmup 3 --variant $v --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_C4_$v.json 2> gpurun_out/r2e_bench_C4_$v.err
done
