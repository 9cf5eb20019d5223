# fast GPU loop: parity suite without the full-size cfg 5 every-row test and the fuzz sweep, then phase times at cfg 2 and 5
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not every_row and not fuzz" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in 2 5; do timeout 300 python tools/run_case.py --config $c --reps 3 > gpurun_out/case$c.json 2>&1; done
