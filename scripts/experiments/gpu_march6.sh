mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for v in cur p1 p3 p6; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  echo "$v $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config 7pt768 2>&1 >/dev/null | tail -1 | cut -c1-110)"
done
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spmv_march" -s 3 -c 1 -o gpurun_out/prof_march768b -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong --config 7pt768 > /dev/null 2>&1; echo "ncu full rc $?"
