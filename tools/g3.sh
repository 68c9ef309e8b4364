mkdir -p gpurun_out
(
timeout 120 python -u tools/prof_train.py --config C4 --K 1024 --rows 1024 --reps 3 2>&1 | tail -1
PNN_RESIDENT_GROUPS=2 timeout 120 python -u tools/prof_train.py --config C4 --K 1024 --rows 1024 --reps 3 2>&1 | tail -1
timeout 60 python -u tools/trace_resident.py --config C4 --K 1 --rows 256 2>&1 | tail -19
timeout 300 python -u -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
) > gpurun_out/g3.log 2>&1
cat gpurun_out/g3.log
