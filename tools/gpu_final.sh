# end-of-round refresh: parity tests, bench line, launch list, ncu of the walk kernels,
# sweeps, symmetric / density / partition timings (all at cfg 5 unless noted)
mkdir -p gpurun_out
bash tools/gpu_bench.sh
bash tools/gpu_ncu_k.sh "walk_kernel|fill_kernel|desc_kernel" 5 3
bash tools/gpu_sym.sh
timeout 300 python tools/density_case.py --config 5 > gpurun_out/density_cfg5.json 2>&1
timeout 300 python tools/density_case.py --config 2 > gpurun_out/density_cfg2.json 2>&1
timeout 600 python tools/part_case.py --config 5 --out gpurun_out/part_cfg5.json > gpurun_out/part.log 2>&1
bash tools/gpu_sweep.sh
