#!/bin/bash
# Round-1 session D GPU batch: full gpu tests, f-row experiments (short), F1/C5 bench.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d_pytest.log
tail -3 gpurun_out/d_pytest.log
timeout 300 python bench.py --config F1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d_bench_F1.json 2> gpurun_out/d_bench_F1.err; tail -c 600 gpurun_out/d_bench_F1.json
timeout 300 python tools/experiments.py table2 > gpurun_out/d_table2.jsonl 2>&1; cat gpurun_out/d_table2.jsonl | cut -c1-200
timeout 600 python tools/experiments.py curves --K 1,2,10 --epochs 3 > gpurun_out/d_curves.jsonl 2>&1; tail -3 gpurun_out/d_curves.jsonl | cut -c1-300
