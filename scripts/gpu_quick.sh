# quick GPU iteration: parity subset + headline bench (fused & unfused)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv or cg_vs or golden or headline" > gpurun_out/pytest_quick.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/pytest_quick.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?; tail -1 gpurun_out/bench.err
timeout 300 python bench.py --steps 5 --warmup 3 --mode unfused --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_unfused.json 2> gpurun_out/bench_unfused.err; tail -1 gpurun_out/bench_unfused.err
