# ncu --set full of kernels matching regex $1 (first $3 launches, default 1) at config $2 (default 5)
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"$1" -c ${3:-1} \
  -o gpurun_out/k_full -f python tools/run_case.py --config ${2:-5} --reps 1 > gpurun_out/ncu_k.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k.log
