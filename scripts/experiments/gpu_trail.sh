# trailing-band L2 prefetch A/B at 768^3 and 512^3 / 256^3 (abvar/trail = with, notrail = without)
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in trail notrail; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  for c in 7pt768 7pt512 7pt256; do
    echo "$c $v $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config $c 2>&1 >/dev/null | tail -1 | cut -c1-110)"
  done
done; done
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
