# GPU check: parity suite, then phase timings at cfg 5 / cfg 2 (gather; cfg 5 also symmetric and tree order)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/chk_tests.log
for c in 5 2; do timeout 300 python tools/run_case.py --config $c --reps 3 > gpurun_out/chk_c$c.json 2>&1; done
timeout 300 python tools/run_case.py --config 5 --reps 3 --symmetric > gpurun_out/chk_sym5.json 2>&1
timeout 300 python tools/run_case.py --config 5 --reps 3 --tree-order > gpurun_out/chk_to5.json 2>&1
timeout 600 python tools/density_case.py --config 5 > gpurun_out/chk_den5.json 2>&1
