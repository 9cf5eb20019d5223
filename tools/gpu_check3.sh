# GPU check: parity suite, gather / symmetric timings at cfg 5 (per-rep phases)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/chk_tests.log
timeout 300 python tools/run_case.py --config 5 --reps 3 > gpurun_out/ab_gather_r1.json 2>&1
timeout 300 python tools/run_case.py --config 5 --reps 3 --symmetric > gpurun_out/ab_sym_r1.json 2>&1
