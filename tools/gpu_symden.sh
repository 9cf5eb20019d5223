# symmetric + density: parity tests, then timings at cfg 2 and 5
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "symmetric or density or sym or fuzz or partition or fill_only" > gpurun_out/gpu_tests_symden.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_symden.log
for c in 2 5; do timeout 600 python tools/density_case.py --config $c > gpurun_out/density_cfg$c.json 2>&1; done
for c in 2 5; do timeout 600 python tools/run_case.py --config $c --reps 3 --symmetric > gpurun_out/sym_cfg$c.json 2>&1; done
