# A/B of libbtree_*.so variants at cfg 5 in caller order and tree order (results under gpurun_out/ab_caller, ab_tree)
mkdir -p gpurun_out
bash tools/gpu_ab.sh 5
mkdir -p gpurun_out/ab_caller; rm -f gpurun_out/ab_caller/*; mv gpurun_out/ab_*_r*.json gpurun_out/ab_caller/
bash tools/gpu_ab.sh 5 --tree-order
mkdir -p gpurun_out/ab_tree; rm -f gpurun_out/ab_tree/*; mv gpurun_out/ab_*_r*.json gpurun_out/ab_tree/
