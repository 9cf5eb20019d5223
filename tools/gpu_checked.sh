# the GPU parity + fuzz suites against the bounds-checked build (-DBT_CHECKED:
# device-side index checks trap on any out-of-range access)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DBT_CHECKED \
  paper_1910_02639_b200/csrc/*.cu -o paper_1910_02639_b200/libbtree_checked.so > gpurun_out/checked_build.log 2>&1
BT_LIB=$PWD/paper_1910_02639_b200/libbtree_checked.so timeout 1500 python -m pytest tests -m gpu -q -k "not every_row" \
  > gpurun_out/checked_tests.log 2>&1
echo "checked tests rc=$?" >> gpurun_out/checked_tests.log
