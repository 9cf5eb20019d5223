# parity suite on the in-tree library, then tools/gpu_ab.sh on the variants ($1: config, $2: run_case flags)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/chk_tests.log
bash tools/gpu_ab.sh ${1:-5} "${2:-}"
