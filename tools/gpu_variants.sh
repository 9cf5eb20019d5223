# time the search at config $1 (default 5) for each library variant paper_1910_02639_b200/libbtree_*.so ($2: extra run_case flags)
mkdir -p gpurun_out
for f in paper_1910_02639_b200/libbtree_*.so; do
  v=$(basename $f .so)
  BT_LIB=$PWD/$f timeout 300 python tools/run_case.py --config ${1:-5} --reps 3 ${2:-} > gpurun_out/var_${v}_c${1:-5}.json 2>&1
done
