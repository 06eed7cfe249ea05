# ncu --set full of one K1 launch for each prebuilt library variant abvar/<name>/librvk.so
mkdir -p gpurun_out
for v in "$@"; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/ab_k1_$v -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $v rc $?"
done
