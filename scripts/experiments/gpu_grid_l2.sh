# L2 grid solve (k_cg_grid_l2, RVK_PLAN_GRID_L2): parity tests, then AUTO
# (grid L2) vs the fused graph on the sizes it covers
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_grid_solve.py -q -x -p no:cacheprovider > gpurun_out/pytest_grid.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_grid.log
for c in 5pt512 5pt768 5pt1024 9pt1024 7pt100; do
  echo "$c auto  $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode auto 2>&1 >/dev/null | tail -1 | cut -c1-70)"
  echo "$c fused $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode fused 2>&1 >/dev/null | tail -1 | cut -c1-70)"
done
