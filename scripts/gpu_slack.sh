mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tfqmr.py -x -q > gpurun_out/pytest_slack.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_slack.log
for c in 27pt256 7pt256 9pt4096; do for sl in 1 0; do
  RVK_SPMV_SLACK=$sl timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config $c > /dev/null 2> gpurun_out/b_${c}_$sl.err; echo "$c slack=$sl $(tail -1 gpurun_out/b_${c}_$sl.err)"
done; done
RVK_SPMV_SLACK=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config 27pt256 --solver tfqmr > /dev/null 2> gpurun_out/b_tfq27.err; echo "tfqmr 27 $(tail -1 gpurun_out/b_tfq27.err)"
