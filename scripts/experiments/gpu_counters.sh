# incremental stage/phase counters + tile via stage meta (abvar/n1 row order, n2 = 2 chunks/plane) vs old
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in n3 n1 old; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  for c in 7pt256 27pt256 9pt4096 7pt768; do
    echo "$c $v $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config $c 2>&1 >/dev/null | tail -1 | cut -c1-90)"
  done
done; done
cp abvar/n3/librvk.so paper_2306_17801_b200/lib/librvk.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_tfqmr.py -q -x -p no:cacheprovider 2>&1 | tail -2
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
