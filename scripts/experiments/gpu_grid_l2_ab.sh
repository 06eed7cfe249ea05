# A/B of grid-solve library variants (abvar/<name>/librvk.so), then the grid
# tests on the last one (= the in-tree build)
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_intree.so
CFGS="${CFGS:-5pt256 5pt512 5pt768 5pt1024}" ROUNDS=${ROUNDS:-1} bash scripts/experiments/ab_libs.sh "$@"
cp /tmp/librvk_intree.so paper_2306_17801_b200/lib/librvk.so
timeout 600 python -m pytest tests/test_gpu_grid_solve.py -q -x -p no:cacheprovider > gpurun_out/pytest_grid.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_grid.log
