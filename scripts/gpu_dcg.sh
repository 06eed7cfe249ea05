exec > gpurun_out/dcg.log 2>&1
for c in 5pt256 5pt512 5pt1024; do
for sr in 0 524288; do
RVK_SMALL_ROWS=$sr timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $c --mode fused 2>&1 >/dev/null | tail -1 | sed "s/^/$c small=$sr /" | cut -c1-110
done; done
