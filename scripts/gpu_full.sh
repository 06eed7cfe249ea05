# Full measurement pass: all configs + ncu launch list + ncu --set full of K1/K2.
mkdir -p gpurun_out
for c in 7pt256 27pt256 9pt4096 5pt1024 5pt64 5pt128 5pt256 5pt512; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc $? $(tail -1 gpurun_out/bench_$c.err)"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 123 -c 82 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu launches rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k1.log 2>&1; echo ncu k1 rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_update -s 4 -c 1 -o gpurun_out/prof_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k2.log 2>&1; echo ncu k2 rc $?
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1_27pt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config 27pt256 > /dev/null 2>&1; echo ncu k1 27pt rc $?
