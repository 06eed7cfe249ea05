# latency sweep: persistent vs fused graph vs host-sync baseline (2D 5-pt 64^2..1024^2)
mkdir -p gpurun_out
for c in 5pt64 5pt128 5pt256 5pt512 5pt1024; do
  for m in persistent fused hostsync; do
    timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --config $c --mode $m > gpurun_out/sweep_${c}_${m}.json 2> gpurun_out/sweep_${c}_${m}.err
    echo "$c $m rc $? $(tail -1 gpurun_out/sweep_${c}_${m}.err)"
  done
done
