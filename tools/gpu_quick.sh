# quick GPU check: parity tests + phase timings at cfg 2..5
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in 2 3 4 5; do timeout 300 python tools/run_case.py --config $c --reps 3 > gpurun_out/case$c.json 2>&1; done
