exec > gpurun_out/dcg.log 2>&1
timeout 600 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -x -q -k "api or cluster or small or golden or oracle" 2>&1 | tail -2
for c in 5pt64 5pt256 5pt512 5pt1024 7pt256; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $c 2>&1 >/dev/null | tail -1 | sed "s/^/$c auto /" | cut -c1-100
done
