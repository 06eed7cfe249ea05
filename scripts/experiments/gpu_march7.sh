# march K1 without per-tile divisions vs row order (RVK_OPT_MARCH = 1024)
mkdir -p gpurun_out
for r in 1 2; do for o in 1024 0; do for c in 7pt768 7pt512; do
  echo "$c opts=$o $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config $c --opts $o 2>&1 >/dev/null | tail -1 | cut -c1-100)"
done; done; done
timeout 900 python -m pytest tests/test_gpu_march.py -q -p no:cacheprovider 2>&1 | tail -2
