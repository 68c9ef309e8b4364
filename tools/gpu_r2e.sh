#!/bin/bash
# quick v12 check: parity subset, C4 bench, trace
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ws or short" > gpurun_out/r2e_pytest_ws.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2e_pytest_ws.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_C4_ws.json 2> gpurun_out/r2e_bench_C4_ws.err
PNN_LIB=$PWD/paper_2304_09590_b200/libpnn_tr.so timeout 300 python tools/trace_ws.py > gpurun_out/r2e_trace.txt 2>&1
