# probe: random-order CSR row writes (tools/probe_rows.cu) + one cfg 5 bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/probe_rows.log 2>&1
timeout 300 ./tools/probe_rows >> gpurun_out/probe_rows.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err
