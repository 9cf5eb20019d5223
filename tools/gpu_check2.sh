# GPU check: parity suite, phase timings at cfg 5 / cfg 2, library variants at cfg 5
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/chk_tests.log
for c in 5 2; do timeout 300 python tools/run_case.py --config $c --reps 3 > gpurun_out/chk_c$c.json 2>&1; done
bash tools/gpu_variants.sh 5
