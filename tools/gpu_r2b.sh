# full parity suite, then gather / symmetric / density timings at cfg 2 and 5
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in 2 5; do
  timeout 300 python tools/run_case.py --config $c --reps 3 > gpurun_out/case$c.json 2>&1
  timeout 300 python tools/run_case.py --config $c --reps 3 --symmetric > gpurun_out/sym_cfg$c.json 2>&1
  timeout 600 python tools/density_case.py --config $c > gpurun_out/density_cfg$c.json 2>&1
done
