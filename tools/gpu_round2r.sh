#!/bin/bash
# Round-2 closing batch (r) on the final build (Gram pre-pass 0.547 ms): smoke, the default C4 bench line, the full
# GPU suite, the C4 launch list, ncu full captures of the v12 SGD launch and the Gram pre-pass.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-r2r}; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err; echo "bench C4 rc=$?"
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err; echo "bench C3 rc=$?"
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv $B > /dev/null 2>&1; echo "launches C4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_ws -s 3 -c 1 -o $O/prof_ws_C4 $B > $O/ncu.log 2>&1; echo "ncu C4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram -s 3 -c 1 -o $O/prof_gram_C4 $B > $O/ncu_gram.log 2>&1; echo "ncu gram rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
