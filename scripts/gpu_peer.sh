# PEER backend loopback tests + parity subset + headline bench + K2 profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded.log 2>&1; echo "sharded rc $?"; tail -3 gpurun_out/pytest_sharded.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "parity rc $?"; tail -2 gpurun_out/pytest_parity.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc $?"; cat gpurun_out/bench_default.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 123 -c 82 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu launches rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_update -s 4 -c 1 -o gpurun_out/prof_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k2.log 2>&1; echo ncu k2 rc $?
