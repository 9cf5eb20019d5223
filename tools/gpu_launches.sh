# launch list (ncu, serialised) of one run_case call at config $1
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_case.csv python tools/run_case.py --config ${1:-5} --reps 1 ${2:-} > gpurun_out/ncu_case.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_case.log
