mkdir -p gpurun_out
PNN_LIB=paper_2304_09590_b200/libpnn_dbg.so timeout 100 python -u tools/prof_train.py --config C4 --K 1 --rows 64 --reps 1 > gpurun_out/dbg1.log 2>&1; echo rc=$?; tail -5 gpurun_out/dbg1.log
PNN_LIB=paper_2304_09590_b200/libpnn_dbg.so PNN_RESIDENT_GROUPS=2 timeout 100 python -u tools/prof_train.py --config C4 --K 2 --rows 64 --reps 1 > gpurun_out/dbg2.log 2>&1; echo rc=$?; tail -5 gpurun_out/dbg2.log
PNN_LIB=paper_2304_09590_b200/libpnn_dbg.so timeout 300 python -u -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/dbgtest.log 2>&1; echo rc=$?; tail -5 gpurun_out/dbgtest.log
