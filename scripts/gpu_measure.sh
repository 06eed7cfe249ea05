mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --steps 5 --warmup 3 --mode unfused --no-cpu-baseline > gpurun_out/bench_unfused.json 2> gpurun_out/bench_unfused.err; tail -1 gpurun_out/bench_unfused.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k1.log 2>&1; echo ncu2 rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_update -s 4 -c 1 -o gpurun_out/prof_k2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k2.log 2>&1; echo ncu3 rc $?
