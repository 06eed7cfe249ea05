exec > gpurun_out/dcg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or persistent" 2>&1 | tail -4
for c in 5pt64 5pt128 5pt256 5pt512; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $c --mode auto 2>&1 >/dev/null | tail -1 | sed "s/^/$c auto /"
done
