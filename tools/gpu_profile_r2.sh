# round-2 evidence: parity suite, bench line, ncu launch list of one bench step,
# ncu --set full of the search kernels and of the build's scatter / key_hist (cfg 5)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc=$?" >> gpurun_out/ncu_launch.log
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel|fill_kernel|desc_kernel" -c 3 \
  -o gpurun_out/k_full -f python tools/run_case.py --config 5 --reps 1 > gpurun_out/ncu_k.log 2>&1
echo "ncu k rc=$?" >> gpurun_out/ncu_k.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"scatter_kernel|key_hist_kernel|leaf_finalize" -c 3 \
  -o gpurun_out/b_full -f python tools/run_case.py --config 5 --reps 1 > gpurun_out/ncu_b.log 2>&1
echo "ncu b rc=$?" >> gpurun_out/ncu_b.log
