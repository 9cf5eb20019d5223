# fill with per-round prefix packs (BT_FILL_PRE): A/B of libbtree_pre*.so at cfg 5 (caller and tree order) and cfg 2,
# then the parity suite against libbtree_pre1b.so
mkdir -p gpurun_out
bash tools/gpu_ab.sh 5
mkdir -p gpurun_out/ab_caller; rm -f gpurun_out/ab_caller/*; mv gpurun_out/ab_*_r*.json gpurun_out/ab_caller/
bash tools/gpu_ab.sh 5 --tree-order
mkdir -p gpurun_out/ab_tree; rm -f gpurun_out/ab_tree/*; mv gpurun_out/ab_*_r*.json gpurun_out/ab_tree/
bash tools/gpu_ab.sh 2
mkdir -p gpurun_out/ab_cfg2; rm -f gpurun_out/ab_cfg2/*; mv gpurun_out/ab_*_r*.json gpurun_out/ab_cfg2/
BT_LIB=$PWD/paper_1910_02639_b200/libbtree_pre1b.so timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pre_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/pre_tests.log
tail -3 gpurun_out/pre_tests.log
