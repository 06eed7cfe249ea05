mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_xd.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_xd.log
for c in 7pt256 27pt256; do for d in 1 0 1 0; do
RVK_X_DEFER=$d timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > /dev/null 2> /tmp/e.err; echo "$c defer=$d $(tail -1 /tmp/e.err)"
done; done
for d in 1 0; do RVK_X_DEFER=$d timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --operator stencil > /dev/null 2> /tmp/e.err; echo "mf7 defer=$d $(tail -1 /tmp/e.err)"; done
