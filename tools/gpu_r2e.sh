#!/bin/bash
# round 2e: warp-specialised TMEM variant (v12, k_ws.cu): parity + bench; e1 chain-only, e2 sweep-only, e3 = 2 smem rows
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ws" > gpurun_out/r2e_pytest_ws.log 2>&1
echo "pytest ws exit $?" >> gpurun_out/r2e_pytest_ws.log
timeout 300 python bench.py --steps 5 --warmup 3 --variant ws --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_C4_ws.json 2> gpurun_out/r2e_bench_C4_ws.err
for e in e1 e2 e3; do
  PNN_LIB=$PWD/paper_2304_09590_b200/libpnn_$e.so timeout 300 python bench.py --steps 5 --warmup 3 --variant ws --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_C4_ws_$e.json 2> gpurun_out/r2e_bench_C4_ws_$e.err
done
