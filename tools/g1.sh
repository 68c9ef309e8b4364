nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/trace_resident.py --config C4 --K 1 --rows 256 > gpurun_out/trace1.log 2>&1; echo trace=$?
timeout 300 python tools/trace_resident.py --config C4 --K 33 --rows 256 > gpurun_out/trace33.log 2>&1; echo trace33=$?
cat gpurun_out/trace1.log gpurun_out/trace33.log
