# re-entry check: parity suite, smoke, default bench line (cfg 5) from a rebuilt tree
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/re_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/re_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/re_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/re_bench_cfg5.json 2> gpurun_out/re_bench_cfg5.err; echo "bench rc=$?" >> gpurun_out/re_bench_cfg5.err
tail -3 gpurun_out/re_gpu_tests.log; tail -2 gpurun_out/re_smoke.log; tail -2 gpurun_out/re_bench_cfg5.err
