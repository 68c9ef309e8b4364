# quick: parity of resident v4 + timing
timeout 120 python tools/prof_train.py --config C4 --K 1 --rows 1024 --reps 3 2>&1 | tail -2
timeout 120 python tools/prof_train.py --config C4 --K 74 --rows 1024 --reps 3 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1
