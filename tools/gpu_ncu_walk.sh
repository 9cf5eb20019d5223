# ncu --set full of the walk kernels at cfg 5 (one launch each)
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"desc_kernel|walk_kernel|fill_kernel" -c 3 \
  -o gpurun_out/walk_full -f python tools/run_case.py --config 5 --reps 1 > gpurun_out/ncu_walk.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_walk.log
