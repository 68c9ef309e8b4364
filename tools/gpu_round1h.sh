#!/bin/bash
# Round-1 final measurement batch: full GPU tests, smoke, bench lines for every config,
# launch list + ncu full capture of the C4 bench's dominant kernel.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/h_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/h_smoke.log
timeout 900 python bench.py > gpurun_out/h_bench_C4.json 2> gpurun_out/h_bench_C4.err; echo "bench C4 rc=$?"
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/h_bench_ref_C4.json 2>&1; echo "ref rc=$?"
for c in C1 C2 C3 C5 F1; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/h_bench_$c.json 2> gpurun_out/h_bench_$c.err; echo "bench $c rc=$?"; done
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/h_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_launches_C4.csv $B > /dev/null 2>&1; echo "launches rc=$?"
timeout 300 $B > gpurun_out/h_plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_resident -s 3 -c 1 -o gpurun_out/prof_resident_C4_final $B > gpurun_out/h_ncu.log 2>&1; echo "ncu rc=$?"
