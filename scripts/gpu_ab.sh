# A/B: x-windows on/off, parity subset first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_sanitizer.py -x -q > gpurun_out/pytest_ab.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_ab.log
for c in 7pt256 27pt256 9pt4096 5pt1024; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/ab_win_$c.json 2> gpurun_out/ab_win_$c.err; echo "win   $c $(tail -1 gpurun_out/ab_win_$c.err)"
  RVK_NO_WINDOWS=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/ab_nowin_$c.json 2> gpurun_out/ab_nowin_$c.err; echo "nowin $c $(tail -1 gpurun_out/ab_nowin_$c.err)"
done
