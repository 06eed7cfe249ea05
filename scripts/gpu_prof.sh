# bench + ncu full capture of the fused SpMV (K1) and the update kernel (K2)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?; tail -1 gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_k1.log 2>&1; echo ncu k1 rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_update -s 4 -c 1 -o gpurun_out/prof_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_k2.log 2>&1; echo ncu k2 rc $?
