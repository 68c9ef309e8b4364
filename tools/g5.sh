mkdir -p gpurun_out
timeout 120 python tools/prof_train.py --config C4 --K 74 --rows 512 --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_resident -s 1 -c 1 -o gpurun_out/prof_v7 python tools/prof_train.py --config C4 --K 74 --rows 512 --reps 1 > gpurun_out/ncu_v7.log 2>&1
echo ncu=$?
tail -3 gpurun_out/ncu_v7.log
