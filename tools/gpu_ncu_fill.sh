# ncu --set full of the fill kernel of library variant $1 at config ${2:-5}
mkdir -p gpurun_out
v=$1
BT_LIB=$PWD/paper_1910_02639_b200/$v timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fill" -c 1 \
  -o gpurun_out/fill_$v -f python tools/run_case.py --config ${2:-5} --reps 1 > gpurun_out/fill_ncu_$v.log 2>&1
ncu -i gpurun_out/fill_$v.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/fill_src_$v.csv 2>/dev/null
ncu -i gpurun_out/fill_$v.ncu-rep --page details --csv > gpurun_out/fill_det_$v.csv 2>/dev/null
