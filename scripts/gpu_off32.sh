mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_tfqmr.py tests/test_gpu_sanitizer.py -x -q > gpurun_out/pytest_off32.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_off32.log
for c in 7pt256 9pt4096 27pt256; do for o in 1 0; do
RVK_OFF32=$o timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > /dev/null 2> /tmp/e.err; echo "$c off32=$o $(tail -1 /tmp/e.err)"
done; done
