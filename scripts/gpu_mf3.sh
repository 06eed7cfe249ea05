mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "matrix_free or while" > gpurun_out/pytest_mf.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_mf.log
for c in 27pt256 7pt256 9pt4096; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --operator stencil --config $c > /dev/null 2> gpurun_out/mf_$c.err; echo "$c $(tail -1 gpurun_out/mf_$c.err)"
done
