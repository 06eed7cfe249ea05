mkdir -p gpurun_out
timeout 600 ./scripts/probes/tma_stream_probe > gpurun_out/tma_stream_probe.txt 2>&1; echo "probe rc $?"; cat gpurun_out/tma_stream_probe.txt
timeout 1500 python -m pytest tests/test_gpu_march.py -q -p no:cacheprovider > gpurun_out/pytest_march.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/pytest_march.log
for c in 7pt768; do for o in 0 2048; do
  echo "$c opts=$o $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config $c --opts $o 2>&1 >/dev/null | tail -1 | cut -c1-150)"
done; done
timeout 300 python scripts/shard_k1_probe.py
