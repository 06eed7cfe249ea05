exec > gpurun_out/dcg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "persistent" 2>&1 | tail -5
for c in 5pt64 5pt128 5pt256 5pt512; do
for m in auto fused; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $c --mode $m 2>&1 >/dev/null | tail -1 | sed "s/^/$c $m /"
done; done
RVK_CLUSTER=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config 5pt64 --mode persistent 2>&1 >/dev/null | tail -1 | sed "s/^/5pt64 gridbarrier /"
