# early stage release A/B (abvar/er1 = release before the gathers, er0 = after the tile)
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in er1 er0; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  for c in 7pt256 7pt768 9pt4096 5pt1024 27pt256; do
    echo "$c $v $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 10 --warmup 3 --config $c 2>&1 >/dev/null | tail -1 | cut -c1-100)"
  done
done; done
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
