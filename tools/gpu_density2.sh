# density (dense fp32 sum): parity tests + time / error at cfg 2 and 5
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "density or fuzz or partition" > gpurun_out/gpu_tests_density.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_density.log
for c in 2 5; do timeout 600 python tools/density_case.py --config $c > gpurun_out/density_cfg$c.json 2>&1; done
