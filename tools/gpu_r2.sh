# round 2 check: parity suite + per-config phase timings + bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in 2 5; do timeout 300 python tools/run_case.py --config $c --reps 3 > gpurun_out/case$c.json 2>&1; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
