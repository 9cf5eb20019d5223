# ncu --set full of the symmetric walk kernel (walk_kernel<0, 1>) and descent at cfg 5
mkdir -p gpurun_out/sym
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel|desc_kernel" -c 2 \
  -o gpurun_out/sym/sym_full -f python tools/run_case.py --config 5 --reps 1 --symmetric > gpurun_out/sym/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/sym/ncu.log
ncu -i gpurun_out/sym/sym_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/sym/src.csv 2>/dev/null
ncu -i gpurun_out/sym/sym_full.ncu-rep --page details --csv > gpurun_out/sym/det.csv 2>/dev/null
