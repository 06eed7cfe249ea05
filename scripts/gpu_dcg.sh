exec > gpurun_out/dcg.log 2>&1
for h in 0 1 3; do
RVK_L2_HINTS=$h timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config 7pt768 2>&1 >/dev/null | tail -1 | sed "s/^/768 h=$h /"
done
for h in 0 1 3; do
RVK_L2_HINTS=$h timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | tail -1 | sed "s/^/256 h=$h /"
done
