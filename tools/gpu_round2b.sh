#!/bin/bash
# Round-2 batch (b): full GPU tests (incl. slow), smoke, bench lines for every config, the
# reference arm, C5 launch list + ncu full captures of the step kernels (final build).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out/r2b
O=gpurun_out/r2b
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err; echo "bench C4 rc=$?"
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref_C4.json 2>&1; echo "ref rc=$?"
for c in C1 C2 C3 C5 F1; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"; done
timeout 600 python bench.py --variant v8 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4_v8.json 2>&1; echo "bench C4 v8 rc=$?"
B5="python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B5 > $O/plain5.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv $B5 > /dev/null 2>&1; echo "launches C5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|mb_out_bwd|mb_cast_x" -s 60 -c 7 -o $O/prof_c5 python tools/c5_small.py 8 > $O/ncu5.log 2>&1; echo "ncu C5 rc=$?"
timeout 300 python tools/trace_tc.py > $O/trace_tc.log 2>&1; echo "trace rc=$?"
