# pencil tile order A/B (abvar/pencil: planes >= 512^2 walk tile columns through z)
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in pencil row; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  for c in 7pt768 7pt512; do
    echo "$c $v $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config $c 2>&1 >/dev/null | tail -1 | cut -c1-110)"
  done
done; done
cp abvar/pencil/librvk.so paper_2306_17801_b200/lib/librvk.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_spmv" -s 6 -c 2 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong --config 7pt768 > gpurun_out/pencil_ncu.csv 2>/dev/null; echo "ncu rc $?"
timeout 1200 python -m pytest tests/test_gpu_baseline_sizes.py -q -x -p no:cacheprovider -k "768_single" 2>&1 | tail -2
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
