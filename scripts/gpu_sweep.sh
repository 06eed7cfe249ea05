# latency sweep (AUTO vs fused vs host-sync) + the solve-mode tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid_solve.py tests/test_gpu_parity.py tests/test_gpu_api.py -q -p no:cacheprovider > gpurun_out/pytest_sweep.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_sweep.log
for c in 5pt64 5pt128 5pt256 5pt512 5pt768 5pt1024; do
  echo "$c auto  $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode auto 2>&1 >/dev/null | tail -1 | cut -c1-60)"
  echo "$c fused $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode fused 2>&1 >/dev/null | tail -1 | cut -c1-60)"
  echo "$c hostsync $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 10 --warmup 3 --config $c --mode hostsync 2>&1 >/dev/null | tail -1 | cut -c1-60)"
done
