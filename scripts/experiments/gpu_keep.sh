# CSR L2 residency A/B for L2-sized systems (abvar/k0 = evict_first always,
# k100 / k120 = normal priority when the iteration's working set <= 100 / 120 MB)
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in k0 k120 k100; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  for c in 5pt1024 5pt512; do
    echo "$c $v $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 20 --warmup 5 --config $c --mode fused 2>&1 >/dev/null | tail -1 | cut -c1-100)"
  done
done; done
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
