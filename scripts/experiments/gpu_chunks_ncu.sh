mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for v in c1 c2; do
cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spmv_tma" -s 4 -c 1 -o gpurun_out/prof768_$v -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong --config 7pt768 > /dev/null 2>&1; echo "ncu $v rc $?"
done
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
