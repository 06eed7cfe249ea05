# K2 variants at their own resident wave (abvar/new) vs the shared update grid (old)
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in new old; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  for c in 7pt256 27pt256 9pt4096; do
    echo "$c $v $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 10 --warmup 3 --config $c 2>&1 >/dev/null | tail -1 | cut -c1-90)"
  done
  echo "$v $(timeout 300 python scripts/shard_k1_probe.py 2>&1 | tail -1)"
done; done
cp abvar/new/librvk.so paper_2306_17801_b200/lib/librvk.so
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
