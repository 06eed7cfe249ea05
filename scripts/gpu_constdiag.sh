mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_api.py -x -q > gpurun_out/pytest_cd.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_cd.log
for c in 7pt256 27pt256 9pt4096; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/bench_cd_$c.json 2> gpurun_out/bench_cd_$c.err; echo "$c $(tail -1 gpurun_out/bench_cd_$c.err)"
done
