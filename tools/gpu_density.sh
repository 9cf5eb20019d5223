timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "density" > gpurun_out/gpu_tests_new.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_new.log
for c in 5; do timeout 300 python tools/density_case.py --config $c > gpurun_out/density_cfg$c.json 2>&1; done
