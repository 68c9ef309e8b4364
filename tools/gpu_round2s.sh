#!/bin/bash
# Round-2 batch (s): final-build ncu --set full digests of the kernels outside the C4 SGD launch: F1 (mbres), C3 (deep),
# and C4's merge and readout, each after its plain command exited 0.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/r2s; mkdir -p $O
N="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python bench.py --config F1 $N > $O/plain_F1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:mbres -s 3 -c 1 -o $O/prof_mbres_F1 python bench.py --config F1 $N > $O/ncu_F1.log 2>&1; echo "ncu F1 rc=$?"
timeout 300 python bench.py --config F1 $N > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_F1.csv python bench.py --config F1 $N > /dev/null 2>&1; echo "launches F1 rc=$?"
timeout 300 python bench.py --config C3 $N > $O/plain_C3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_deep -s 3 -c 1 -o $O/prof_deep_C3 python bench.py --config C3 $N > $O/ncu_C3.log 2>&1; echo "ncu C3 rc=$?"
timeout 300 python bench.py $N > $O/plain_C4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:'predict|merge' -s 6 -c 2 -o $O/prof_tail_C4 python bench.py $N > $O/ncu_C4.log 2>&1; echo "ncu C4 tail rc=$?"
