mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck python scripts/experiments/march_probe.py 512 512 8 > gpurun_out/march_sanitize.log 2>&1; echo "sanitizer rc $?"; grep -E "flags|hist rel|ERROR SUMMARY" gpurun_out/march_sanitize.log | head -4
timeout 1500 python -m pytest tests/test_gpu_march.py tests/test_gpu_grid_solve.py tests/test_gpu_trace.py -q -p no:cacheprovider > gpurun_out/pytest_march.log 2>&1; echo "pytest rc $?"; tail -8 gpurun_out/pytest_march.log
for c in 7pt768 7pt512; do for o in 0 2048; do
  echo "$c opts=$o $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config $c --opts $o 2>&1 >/dev/null | tail -1 | cut -c1-150)"
done; done
for c in 5pt128 5pt256 5pt512; do for o in 0 4096; do
  echo "$c opts=$o $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 20 --warmup 3 --config $c --mode auto --opts $o 2>&1 >/dev/null | tail -1 | cut -c1-120)"
done; done
