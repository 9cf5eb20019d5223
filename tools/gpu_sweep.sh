# s / beta / octree sweeps at cfg 2 and cfg 5
mkdir -p gpurun_out
for c in 2 5; do
  timeout 900 python tools/sweep.py --config $c --reps 3 --out gpurun_out/sweep_cfg$c.json > gpurun_out/sweep_cfg$c.log 2>&1
  echo "cfg $c rc=$?" >> gpurun_out/sweep_cfg$c.log
done
timeout 900 python tools/sweep.py --plane 16777216 --reps 3 --out gpurun_out/sweep_plane.json > gpurun_out/sweep_plane.log 2>&1
echo "plane rc=$?" >> gpurun_out/sweep_plane.log
