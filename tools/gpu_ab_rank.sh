# build variant BT_RANK_HIST: parity suite against libbtree_rank.so, then A/B of libbtree_*.so at cfg 5 and cfg 4
mkdir -p gpurun_out/abr
BT_LIB=$PWD/paper_1910_02639_b200/libbtree_rank.so timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/abr/rank_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/abr/rank_tests.log
for c in 5 4; do
  bash tools/gpu_ab.sh $c
  mkdir -p gpurun_out/abr/cfg$c; mv gpurun_out/ab_*_r*.json gpurun_out/abr/cfg$c/
done
