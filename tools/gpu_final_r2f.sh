# round-2 closing captures after the fill's per-round prefix packs (BT_FILL_PRE): launch lists cfg 2-5,
# ncu --set full of the search kernels at cfg 5 / cfg 2 and of the tree-order fill
mkdir -p gpurun_out/final10
O=gpurun_out/final10
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg5.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-tree-order > $O/ncu_launch.log 2>&1
for c in 2 3 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_cfg$c.csv python tools/run_case.py --config $c --reps 1 > $O/ncu_launch_cfg$c.log 2>&1
done
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel|fill_kernel|desc_kernel" -c 3 \
  -o $O/k_full -f python tools/run_case.py --config 5 --reps 1 > $O/ncu_k.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel|fill_kernel|desc_kernel" -c 3 \
  -o $O/k2_full -f python tools/run_case.py --config 2 --reps 1 > $O/ncu_k2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fill_kernel" -c 1 \
  -o $O/fill_to -f python tools/run_case.py --config 5 --reps 1 --tree-order > $O/ncu_fill_to.log 2>&1
ls -la $O
