mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv or cg_vs or golden or chunked or xwindow" > gpurun_out/pytest_pair.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_pair.log
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_tfqmr.py -x -q > gpurun_out/pytest_pair2.log 2>&1; echo "pytest2 rc $?"; tail -2 gpurun_out/pytest_pair2.log
for c in 27pt256; do for pr in 1 0; do
RVK_DEBUG=1 RVK_SPMV_PAIR=$pr timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > /dev/null 2> /tmp/e.err; echo "$c pair=$pr $(grep -o 'R=[0-9]* stages=[0-9]* groups=[0-9]*' /tmp/e.err | head -1) $(tail -1 /tmp/e.err)"
done; done
RVK_SPMV_PAIR=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config 27pt256 --solver tfqmr > /dev/null 2> /tmp/e.err; echo "tfqmr27 $(tail -1 /tmp/e.err)"
