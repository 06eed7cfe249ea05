mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "solve_host_many or cg_vs_oracle or while" > gpurun_out/pytest_many.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_many.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc $?"; cat gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default.err
