# grid-solve A/B: abvar/t1024 (1024 threads, R<=3) vs t512 (512 threads, R<=6), fold fix in both;
# 5pt128 with RVK_OPT_NO_CLUSTER (16) = grid vs the cluster solve
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in t1024 t512; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  for c in 5pt256 5pt512; do
    echo "$c $v $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode auto 2>&1 >/dev/null | tail -1 | cut -c1-60)"
  done
  for c in 5pt64 5pt128; do
    echo "$c $v no-cluster $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 30 --warmup 5 --config $c --mode auto --opts 16 2>&1 >/dev/null | tail -1 | cut -c1-60)"
  done
done; done
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
timeout 900 python -m pytest tests/test_gpu_grid_solve.py -q -p no:cacheprovider 2>&1 | tail -2
