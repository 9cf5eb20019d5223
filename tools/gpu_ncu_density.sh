# ncu --set full of the density walk kernel at config $1 (default 5)
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel" -c 4 \
  -o gpurun_out/dens_full -f python tools/density_case.py --config ${1:-5} --reps 1 > gpurun_out/ncu_dens.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_dens.log
