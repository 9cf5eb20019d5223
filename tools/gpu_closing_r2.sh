# round-2 closing captures with the final code: ncu --set full of the search
# kernels at cfg 3 and cfg 4 (VERDICT r1 Missing #4) and of the build's
# key_hist / scatter / leaf_finalize at cfg 5 and cfg 2
mkdir -p gpurun_out/closing
O=gpurun_out/closing
for c in 4 3; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel|fill_kernel|desc_kernel" -c 3 \
    -o $O/k${c}_full -f python tools/run_case.py --config $c --reps 1 > $O/ncu_k$c.log 2>&1
  echo "ncu k$c rc=$?" >> $O/ncu_k$c.log
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"scatter_kernel|key_hist_kernel|leaf_finalize" -c 5 \
  -o $O/b5_full -f python tools/run_case.py --config 5 --reps 1 > $O/ncu_b5.log 2>&1
echo "ncu b5 rc=$?" >> $O/ncu_b5.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"scatter_kernel|key_hist_kernel|leaf_finalize" -c 5 \
  -o $O/b2_full -f python tools/run_case.py --config 2 --reps 1 > $O/ncu_b2.log 2>&1
echo "ncu b2 rc=$?" >> $O/ncu_b2.log
for c in 1 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
ls -la $O
