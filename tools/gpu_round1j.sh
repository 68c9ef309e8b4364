#!/bin/bash
# Round-1 final measurement batch (deep C3 variant, resident mini-batch F1): full GPU tests, smoke, bench
# lines for every config, C4 launch list + ncu full capture of the resident kernel, C3 launch
# list + ncu full capture of the deep kernel.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/j_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/j_smoke.log
timeout 900 python bench.py > gpurun_out/j_bench_C4.json 2> gpurun_out/j_bench_C4.err; echo "bench C4 rc=$?"
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/j_bench_ref_C4.json 2>&1; echo "ref rc=$?"
for c in C1 C2 C3 C5 F1; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/j_bench_$c.json 2> gpurun_out/j_bench_$c.err; echo "bench $c rc=$?"; done
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/j_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_launches_C4.csv $B > /dev/null 2>&1; echo "launches C4 rc=$?"
timeout 300 $B > gpurun_out/j_plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_resident -s 3 -c 1 -o gpurun_out/prof_resident_C4_j $B > gpurun_out/j_ncu.log 2>&1; echo "ncu C4 rc=$?"
B3="python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B3 > gpurun_out/j_plain3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_launches_C3.csv $B3 > /dev/null 2>&1; echo "launches C3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_deep -s 3 -c 1 -o gpurun_out/prof_deep_C3_j $B3 > gpurun_out/j_ncu3.log 2>&1; echo "ncu C3 rc=$?"
