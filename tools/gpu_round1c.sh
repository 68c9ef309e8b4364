# Round-1 (session 2) measurement of resident v8: GPU tests, bench (C4), launch list, one full ncu capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_r1c.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_r1c.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_r1c.log
timeout 900 python bench.py > gpurun_out/bench_r1c.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_r1c.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_launch.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 120 python tools/prof_train.py --K 74 --rows 256 --reps 1 > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_resident -s 1 -c 1 \
  -o gpurun_out/prof_r1c python tools/prof_train.py --K 74 --rows 256 --reps 1 > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
