# quick A/B of the L2 grid solve: its parity tests, then AUTO on the sizes it covers
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_grid_solve.py -q -x -p no:cacheprovider -k "l2 or eligibility" > gpurun_out/pytest_grid.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_grid.log
for c in ${CFGS:-5pt768 5pt1024 9pt1024 7pt100}; do
  echo "$c auto  $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode auto 2>&1 >/dev/null | tail -1 | cut -c1-70)"
done
