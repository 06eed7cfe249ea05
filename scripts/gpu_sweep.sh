# Latency sweep (2D 5-point, 20 iterations): every mode at every size.
exec > gpurun_out/sweep.log 2>&1
for c in 5pt64 5pt128 5pt256 5pt512 5pt1024; do
for m in auto fused persistent hostsync; do
RVK_CLUSTER=$([ $m = persistent ] && echo 0 || echo 1) timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $c --mode $m 2>&1 >/dev/null | tail -1 | sed "s/^/$c $m /" | cut -c1-60
done; done
