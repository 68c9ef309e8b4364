#!/bin/bash
# round 2f: ncu capture of the v12 SGD launch (full build and sweep-only build)
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 120 python tools/c4_small.py 148 256 ws > gpurun_out/r2f_small.log 2>&1 || exit 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_ws -c 1 -o gpurun_out/r2f_ws python tools/c4_small.py 148 256 ws > gpurun_out/r2f_ncu.log 2>&1
PNN_LIB=$PWD/paper_2304_09590_b200/libpnn_e2.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_ws -c 1 -o gpurun_out/r2f_ws_e2 python tools/c4_small.py 148 256 ws > gpurun_out/r2f_ncu_e2.log 2>&1
