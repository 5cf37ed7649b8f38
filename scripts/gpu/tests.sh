nvidia-smi --query-gpu=name,clocks.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1
echo "pytest rc $?" >> gpurun_out/gputest.log
