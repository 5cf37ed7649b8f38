# Round-end profiles of config C (under gpurun, each after its command ran clean without ncu):
#   launch list of the bench command and one ncu --set full capture of the DAS kernel.
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_C.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc $?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:das_tc_kernel -s 1 -c 1 \
  -o gpurun_out/das_tc_C python scripts/profile_das.py C > gpurun_out/ncu_das_tc.log 2>&1
echo "das_tc rc $?" >> gpurun_out/ncu_das_tc.log
