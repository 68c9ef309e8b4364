#!/bin/bash
# Round-2 closing check (k): smoke, C4 bench line (default AUTO), C4 launch list, v12 trace.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/r2k; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err; echo "bench C4 rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "ws or c4 or C4" > $O/pytest_c4.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_c4.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv $B > /dev/null 2>&1; echo "launches C4 rc=$?"
PNN_LIB=$PWD/paper_2304_09590_b200/libpnn_tr.so timeout 300 python tools/trace_ws.py > $O/trace_ws.txt 2>&1; echo "trace ws rc=$?"
