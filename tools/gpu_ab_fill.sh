# fill variants: parity suite against libbtree_fq.so, then A/B (caller order and tree order) of libbtree_*.so
mkdir -p gpurun_out
BT_LIB=$PWD/paper_1910_02639_b200/libbtree_fq.so timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fq_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fq_tests.log
bash tools/gpu_ab.sh 5
mkdir -p gpurun_out/ab_caller; mv gpurun_out/ab_*_r*.json gpurun_out/ab_caller/
bash tools/gpu_ab.sh 5 --tree-order
mkdir -p gpurun_out/ab_tree; mv gpurun_out/ab_*_r*.json gpurun_out/ab_tree/
