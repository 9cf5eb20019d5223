# symmetric criterion timings (cfg 2, 5) next to the gather ones
mkdir -p gpurun_out
for c in 2 5; do
  timeout 300 python tools/run_case.py --config $c --reps 3 --ngmax 640 > gpurun_out/gather_cfg$c.json 2>&1
  timeout 300 python tools/run_case.py --config $c --reps 3 --ngmax 640 --symmetric > gpurun_out/sym_cfg$c.json 2>&1
done
