# fused persistent solve (k_cg_fp): parity tests, then AUTO (fp) vs the fused graph
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp.py -q -x -p no:cacheprovider > gpurun_out/pytest_fp.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_fp.log
for c in ${CFGS:-5pt1024 9pt1024 7pt100}; do
  echo "$c auto  $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode auto 2>&1 >/dev/null | tail -1 | cut -c1-70)"
  echo "$c fused $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode fused 2>&1 >/dev/null | tail -1 | cut -c1-70)"
done
for c in ${BIG:-7pt256 9pt4096}; do
  echo "$c fp    $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 10 --warmup 3 --config $c --opts 16384 2>&1 >/dev/null | tail -1 | cut -c1-70)"
  echo "$c graph $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 10 --warmup 3 --config $c 2>&1 >/dev/null | tail -1 | cut -c1-70)"
done
