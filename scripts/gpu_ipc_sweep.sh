mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer_ipc.py -x -q > gpurun_out/pytest_ipc.log 2>&1; echo "ipc rc $?"; tail -15 gpurun_out/pytest_ipc.log
for c in 27pt256 9pt4096 5pt1024 7pt768; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc $?"; tail -1 gpurun_out/bench_$c.err
done
