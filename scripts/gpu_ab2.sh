# A/B: leading-edge L2 prefetch on/off
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cg_vs or golden or headline or xwindow" > gpurun_out/pytest_ab.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/pytest_ab.log
for c in 7pt256 27pt256 9pt4096 5pt1024; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c 2>&1 >/dev/null | tail -1 | sed "s/^/pf   $c /"
  RVK_NO_PREFETCH=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c 2>&1 >/dev/null | tail -1 | sed "s/^/nopf $c /"
done
