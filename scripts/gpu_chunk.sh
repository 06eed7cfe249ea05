mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "chunked or cg_vs_oracle" > gpurun_out/pytest_chunk.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_chunk.log
for mb in 1000000 80 40 20; do
  RVK_DEBUG=1 RVK_CHUNK_MB=$mb timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config 7pt768 > gpurun_out/bench_768_$mb.json 2> gpurun_out/bench_768_$mb.err; echo "768 mb=$mb rc $? $(grep -o 'order=[^ ]*' gpurun_out/bench_768_$mb.err | head -1) $(tail -1 gpurun_out/bench_768_$mb.err)"
done
RVK_CHUNK_MB=20 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config 27pt256 2> gpurun_out/b27.err > /dev/null; echo "27pt mb=20 $(tail -1 gpurun_out/b27.err)"
