mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_tfqmr.py -x -q > gpurun_out/pytest_unroll.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_unroll.log
for c in 9pt4096 7pt256 27pt256 5pt1024; do for u in 1 8; do
RVK_SPMV_UNROLL=$u timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > /dev/null 2> /tmp/e.err; echo "$c unroll=$u $(tail -1 /tmp/e.err)"
done; done
