#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/e_pytest.log
tail -8 gpurun_out/e_pytest.log
timeout 300 python bench.py --config F1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e_bench_F1.json 2> gpurun_out/e_bench_F1.err; tail -c 900 gpurun_out/e_bench_F1.json
timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e_bench_C5.json 2> gpurun_out/e_bench_C5.err; head -c 300 gpurun_out/e_bench_C5.json
