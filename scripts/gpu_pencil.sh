mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pencil or cg_vs_oracle or spmv" > gpurun_out/pytest_pencil.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_pencil.log
for c in 7pt768 7pt256 27pt256 9pt4096; do for o in row pencil; do
  RVK_TILE_ORDER=$o timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/bench_${c}_$o.json 2> gpurun_out/bench_${c}_$o.err; echo "$c $o rc $? $(tail -1 gpurun_out/bench_${c}_$o.err)"
done; done
