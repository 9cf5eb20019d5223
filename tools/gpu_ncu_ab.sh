# ncu --set full of walk_kernel for two library variants ($1, $2 under paper_1910_02639_b200/) at config $3 (default 5)
mkdir -p gpurun_out
for v in $1 $2; do
  BT_LIB=$PWD/paper_1910_02639_b200/$v timeout 900 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel" -c 1 \
    -o gpurun_out/ab_$v -f python tools/run_case.py --config ${3:-5} --reps 1 > gpurun_out/ab_ncu_$v.log 2>&1
  ncu -i gpurun_out/ab_$v.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ab_src_$v.csv 2>/dev/null
  ncu -i gpurun_out/ab_$v.ncu-rep --page details --csv > gpurun_out/ab_det_$v.csv 2>/dev/null
done
