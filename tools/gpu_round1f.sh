#!/bin/bash
# Round-1 session F: smoke, full C4 bench line, launch list, ncu full captures (resident, a10 GEMMs, f1).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench_C4.json 2> gpurun_out/f_bench_C4.err; echo "bench rc=$?"; tail -c 400 gpurun_out/f_bench_C4.json
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/f_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_C4.csv $B > /dev/null 2>&1; echo "launches rc=$?"
R="python tools/trace_resident.py --config C4 --K 148 --rows 256"
timeout 120 python tools/f1_small.py > gpurun_out/f_f1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:f32_ -s 8 -c 4 -o gpurun_out/prof_f1 python tools/f1_small.py > /dev/null 2>&1; echo "ncu f1 rc=$?"
timeout 120 python tools/c5_small.py 4 > gpurun_out/f_c5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 12 -c 5 -o gpurun_out/prof_c5gemm python tools/c5_small.py 4 > /dev/null 2>&1; echo "ncu c5 rc=$?"
timeout 120 python tools/c5_small.py 4 > gpurun_out/f_c5b.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:mb_ -s 6 -c 5 -o gpurun_out/prof_c5mb python tools/c5_small.py 4 > /dev/null 2>&1; echo "ncu c5mb rc=$?"
ls -la gpurun_out/*.ncu-rep
